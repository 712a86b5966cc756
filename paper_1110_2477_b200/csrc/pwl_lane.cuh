// pwl_lane.cuh -- the per-lane (sequential) node update of the seller / buyer
// recursion, fused into two streaming passes.
//
// One node (Sec. 3): with U = z_{t+1,j}, D = z_{t+1,j+1} (discounted
// to t = 0, see pwl_device.cuh),
//   W = max(U, D)                                  ("w_t"; the /r is the discount)
//   V = W restricted to slopes [lo, hi]            ("v_t"; reading A7:
//       V(y) = inf_y' W(y') + cost of trading y -> y' at the quotes)
//   Z = max(u, V) (seller) / min(u, V) (buyer)
// The restriction is computed as two monotone passes (reading A7):
//   A(y) = inf_{y' >= y} W(y') + lo (y - y')      (buying is the only way up)
//   V(y) = inf_{y' <= y} A(y') + hi (y - y')      (selling is the only way down)
//
// Pass 1 walks right to left: it generates the vertices of W by a merge of U
// and D and feeds them straight into the pass-A recurrence, which writes A
// (reversed) into the lane's scratch.  Pass 2 walks A left to right, runs the
// pass-B recurrence and the envelope with the exercise function u, and writes
// Z straight into its destination.  W and V are never stored.
//
// Every slope is a copy of a value produced once (a quote or a tail), so
// "same slope" is a bitwise test; values closer than ftol() tie and pieces
// shorter than xtol() fold (reading A10 in DESIGN.md; pwl_device.cuh).
#pragma once
#include "pwl_device.cuh"

namespace amtc {

// reversed emitter of pass A (writes buf[(cap-1-m) * stride]); folds
// (near) zero-length pieces into the vertex on their right
template <int STR = 0>
struct RevOutT {
    Vtx* buf;
    int m, cap, stride, err;
    AMTC_HD Vtx& at(int i) { return buf[i * (STR ? STR : stride)]; }
    AMTC_HD void push(double x, double f, double s_right) {
        if (m > 0 && !(x < at(cap - m).x - xtol(x))) return;
        if (m >= cap) { err |= DEV_OVERFLOW; return; }
        Vtx& o = at(cap - 1 - m);
        o.x = x; o.f = f; o.s = s_right;
        m++;
    }
};

// pass-A recurrence, fed W's vertices right to left:
//   push(x, f, sL): W has a vertex at x with value f and slope sL on its left.
// State: tracking (A = W) or flat (A = the line of slope lo through (Lx, Lf)).
// A crossing back to W found while flat lies on W's piece left of x; it is
// confirmed only when the next vertex to the left (or the left tail) shows it
// lies inside that piece.
template <int STR = 0>
struct PassAT {
    double lo;
    double cur_s;          // A's slope just right of the current position
    bool flat;
    double Lx, Lf;         // flat line anchor
    bool pend;             // pending crossing at (yc, fc), after which A follows W with slope ps
    double yc, fc, ps;
    RevOutT<STR> out;

    AMTC_HD void init(double lo_, double right_tail, Vtx* buf, int cap, int stride) {
        lo = lo_; cur_s = right_tail; flat = false; pend = false;
        out.buf = buf; out.m = 0; out.cap = cap; out.stride = stride; out.err = DEV_OK;
    }
    AMTC_HD void resolve(double x_next) {  // x_next: the next W vertex to the left (-inf: none)
        if (!pend) return;
        pend = false;
        if (yc > x_next) {                 // the crossing lies inside the piece
            out.push(yc, fc, lo);
            flat = false;
            cur_s = ps;
        }
    }
    AMTC_HD void push(double x, double fw, double sp) {
        resolve(x);
        double Ax, s_left;
        if (!flat) {
            Ax = fw;
            if (sp >= lo) {
                s_left = sp;
            } else {
                flat = true; Lx = x; Lf = fw; s_left = lo;
            }
        } else {
            Ax = fma(lo, x - Lx, Lf);
            s_left = lo;
            if (sp > lo) {
                const double d = fw - Ax;
                if (d <= ftol(fw, Ax)) {  // W touches the flat line at x: follow W from here
                    flat = false; Ax = fw; s_left = sp;
                } else {
                    pend = true;
                    yc = x - d / (sp - lo);
                    fc = fma(lo, yc - Lx, Lf);
                    ps = sp;
                }
            }
        }
        if (s_left != cur_s) out.push(x, Ax, cur_s);
        cur_s = s_left;
    }
    // left tail of W reached; x0 = W's leftmost vertex (for the anchor of a line)
    AMTC_HD void finish(double x0, double f0) {
        resolve(-INFINITY);
        if (out.m == 0) out.push(x0, flat ? fma(lo, x0 - Lx, Lf) : f0, cur_s);
    }
};

// Pass 1: W = max(U, D) right to left, streamed into pass A.
// Returns DEV_OK / DEV_OVERFLOW / DEV_UNBOUNDED; A = buf[(cap-nA)..cap) (stride),
// with left-tail slope slA.
template <int SO = 0, int SI = 0>
AMTC_HD int lane_pass1(const FnT<SI>& U, const FnT<SI>& D, double lo, Vtx* buf, int cap, int stride, int& nA,
                       double& slA) {
    // current pieces: piece p of F starts at vertex p (p = -1: the left tail)
    int pU = U.n - 1, pD = D.n - 1;
    double axU = U.v(pU).x, afU = U.v(pU).f, sU = U.v(pU).s;
    double axD = D.v(pD).x, afD = D.v(pD).f, sD = D.v(pD).s;
    // winner at +inf: the larger right-tail slope (max); parallel -> larger value
    bool curU;
    if (sU != sD) curU = sU > sD;
    else {
        const double xr = fmax(axU, axD);
        curU = fma(sU, xr - axU, afU) >= fma(sD, xr - axD, afD);
    }
    const double sRt = curU ? sU : sD;  // W's right tail
    if (sRt < lo) { nA = 0; return DEV_UNBOUNDED; }  // restriction infimum is -inf (needs d < r < u)
    PassAT<SO> pa;
    pa.init(lo, sRt, buf, cap, stride);
    double s_pass = sRt;              // W's slope left of the last vertex handed to pass A
    double xlast = 0.0, flast = 0.0;  // that vertex (anchor of a line)
    bool any = false;
    // hand W's vertex (x, f) with left slope sL to pass A (non-kinks are skipped)
    auto wpush = [&](double x, double f, double sL) {
        if (sL != s_pass) {
            pa.push(x, f, sL);
            s_pass = sL;
            xlast = x; flast = f; any = true;
        }
    };
    double x_hi = INFINITY;
    for (;;) {
        const double xa = pU >= 0 ? axU : -INFINITY;
        const double xb = pD >= 0 ? axD : -INFINITY;
        const double x_lo = fmax(xa, xb);
        if (x_lo == -INFINITY) {
            // both on their left tails: the smaller slope wins at -inf
            const bool lU = (sU != sD) ? (sU < sD) : curU;
            if (lU != curU) {  // crossing on (-inf, x_hi)
                const double e_c = curU ? fma(sU, x_hi - axU, afU) : fma(sD, x_hi - axD, afD);
                const double e_o = curU ? fma(sD, x_hi - axD, afD) : fma(sU, x_hi - axU, afU);
                const double s_c = curU ? sU : sD, s_o = curU ? sD : sU;
                double y = x_hi - (e_c - e_o) / (s_c - s_o);
                if (!(y <= x_hi)) y = x_hi;
                wpush(y, fma(s_c, y - x_hi, e_c), s_o);
            }
            break;
        }
        // values at x_lo (exact at a vertex)
        const double eU = (xa == x_lo) ? afU : fma(sU, x_lo - axU, afU);
        const double eD = (xb == x_lo) ? afD : fma(sD, x_lo - axD, afD);
        const double tl = ftol(eU, eD);
        // crossing inside (x_lo, x_hi): the current winner lost strictly at x_lo
        const bool lost = curU ? (eD > eU + tl) : (eU > eD + tl);
        if (lost) {
            const double e_c = curU ? eU : eD, e_o = curU ? eD : eU;
            const double s_c = curU ? sU : sD, s_o = curU ? sD : sU;
            double y = (s_c != s_o) ? x_lo + (e_o - e_c) / (s_c - s_o) : x_lo;
            y = fmin(fmax(y, x_lo), x_hi);
            if (y > x_lo) wpush(y, fma(s_c, y - x_lo, e_c), s_o);
            curU = !curU;
        }
        // step the pointers whose vertex sits at x_lo
        if (xa == x_lo) {
            --pU;
            const Vtx& v = U.v(pU < 0 ? 0 : pU);
            axU = v.x; afU = v.f; sU = pU < 0 ? U.sl : v.s;
        }
        if (xb == x_lo) {
            --pD;
            const Vtx& v = D.v(pD < 0 ? 0 : pD);
            axD = v.x; afD = v.f; sD = pD < 0 ? D.sl : v.s;
        }
        // winner just left of x_lo: by value, ties by the smaller left slope
        if (fabs(eU - eD) > tl) curU = eU > eD;
        else if (sU != sD) curU = sU < sD;
        wpush(x_lo, fmax(eU, eD), curU ? sU : sD);
        x_hi = x_lo;
    }
    if (!any) {  // W is a single line: anchor it at the right-most vertex
        xlast = fmax(U.v(U.n - 1).x, D.v(D.n - 1).x);
        flast = fmax(piece_at(U, U.n - 1, xlast), piece_at(D, D.n - 1, xlast));
    }
    pa.finish(xlast, flast);
    nA = pa.out.m;
    slA = pa.cur_s;
    return pa.out.err;
}

// envelope of V (streamed left to right) with the exercise function u
// (vertex (ux, uf), slopes lo | hi); V's left tail slope is lo as well.
template <int STR = 0>
struct EnvUT {
    bool is_max;
    double ux, uf, lo, hi;
    bool u_passed;       // the current position is right of ux
    double vx, vf, vs;   // current V piece: anchor and slope
    bool curV;           // V is the OP-winner on the current piece
    bool started;
    double x_prev;
    EmitT<STR> E;  // held by value: a pointer would force it into local memory

    AMTC_HD double uval(double y) const { return fma(y < ux ? lo : hi, y - ux, uf); }
    AMTC_HD double su() const { return u_passed ? hi : lo; }
    // an event at xe where V's value is ev (exact when at a V vertex) and u's is eu
    AMTC_HD void event(double xe, double ev, double eu, double new_vs, bool at_u) {
        const double tl = ftol(ev, eu);
        if (!started) {
            // both left tails have slope lo: parallel, the winner is decided by value
            started = true;
            if (fabs(ev - eu) > tl) curV = is_max ? (ev > eu) : (ev < eu);
            else curV = true;
        } else {
            const bool lost = curV ? (is_max ? (eu > ev + tl) : (eu < ev - tl))
                                   : (is_max ? (ev > eu + tl) : (ev < eu - tl));
            if (lost) {
                const double s_c = curV ? vs : su(), s_o = curV ? su() : vs;
                const double e_c = curV ? ev : eu, e_o = curV ? eu : ev;
                double y = (s_c != s_o) ? xe - (e_c - e_o) / (s_c - s_o) : xe;
                y = fmin(fmax(y, x_prev), xe);
                curV = !curV;
                E.push(y, fma(s_o, y - xe, e_o), s_o);
            }
        }
        // pieces right of xe
        if (at_u) u_passed = true;
        vs = new_vs;
        const double s_u = su();
        if (fabs(ev - eu) > tl) curV = is_max ? (ev > eu) : (ev < eu);
        else curV = is_max ? (vs >= s_u) : (vs <= s_u);
        E.push(xe, is_max ? fmax(ev, eu) : fmin(ev, eu), curV ? vs : s_u);
        x_prev = xe;
    }
    // V has a vertex at (x, f) with slope s on its right
    AMTC_HD void push_v(double x, double f, double s) {
        if (!u_passed && ux < x) {  // u's vertex comes first
            event(ux, fma(vs, ux - vx, vf), uf, vs, true);
        }
        const bool at_u = !u_passed && ux == x;
        event(x, f, at_u ? uf : uval(x), s, at_u);
        vx = x; vf = f;
    }
    AMTC_HD void finish() {
        if (!u_passed) event(ux, fma(vs, ux - vx, vf), uf, vs, true);
        // right tails: both have slope hi -> no crossing
    }
};

// Pass 2: V = pass B over A (left to right), Z = OP(u, V) into E.
template <int SE = 0, int SA = 0>
AMTC_HD int lane_pass2(const FnT<SA>& A, double lo, double hi, double ux, double uf, bool seller, EmitT<SE>& Eout) {
    if (A.sl > hi) return DEV_UNBOUNDED;
    EnvUT<SE> env;
    env.E.init(Eout.out, Eout.cap, lo, Eout.stride);
    env.is_max = seller; env.ux = ux; env.uf = uf; env.lo = lo; env.hi = hi;
    env.u_passed = false; env.started = false; env.curV = true;
    env.vx = A.v(0).x; env.vf = A.v(0).f; env.vs = A.sl; env.x_prev = -INFINITY;
    bool flat = false;
    double Mx = 0.0, Mf = 0.0;
    for (int i = 0; i < A.n; ++i) {
        const Vtx& a = A.v(i);
        const double x = a.x, fa = a.f, sp = a.s;  // slope of A right of x
        double Bx, s_right;
        bool cross = false;
        double yc = 0.0, fc = 0.0;
        if (!flat) {
            Bx = fa;
            if (sp <= hi) {
                s_right = sp;
            } else {
                flat = true; Mx = x; Mf = fa; s_right = hi;
            }
        } else {
            Bx = fma(hi, x - Mx, Mf);
            s_right = hi;
            if (sp < hi) {
                const double d = fa - Bx;
                if (d <= ftol(fa, Bx)) {
                    flat = false; Bx = fa; s_right = sp;
                } else {
                    yc = x + d / (hi - sp);
                    if (i + 1 == A.n || yc < A.v(i + 1).x) {
                        cross = true;
                        fc = fma(hi, yc - Mx, Mf);
                    }
                }
            }
        }
#ifndef AMTC_NO_LANE_MERGED
        // one inlined copy of push_v for the vertex and the crossing after it (code size:
        // the solver kernels are instruction-fetch bound)
#pragma unroll 1
        for (int rep = 0; rep < (cross ? 2 : 1); ++rep)
            env.push_v(rep ? yc : x, rep ? fc : Bx, rep ? sp : s_right);
        if (cross) flat = false;
#else
        env.push_v(x, Bx, s_right);
        if (cross) {
            env.push_v(yc, fc, sp);
            flat = false;
        }
#endif
    }
    env.finish();
    env.E.finish();
    Eout = env.E;
    return Eout.err;
}

// the fused node update; scratch: cap vertices at buf (stride); Z -> E
AMTC_HD int lane_node_update(const Fn& U, const Fn& D, double lo, double hi, double ux, double uf, bool seller,
                             Vtx* buf, int cap, int stride, Emit& E) {
    int nA;
    double slA;
    int err = lane_pass1(U, D, lo, buf, cap, stride, nA, slA);
    if (err) return err;
    const Fn A = make_fn(buf + (size_t)(cap - nA) * stride, nA, slA, stride);
    return lane_pass2(A, lo, hi, ux, uf, seller, E);
}

}  // namespace amtc
