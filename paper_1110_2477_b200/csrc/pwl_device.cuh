// pwl_device.cuh -- device-side piecewise-linear (PWL) algebra for the
// Roux-Zastawniak seller/buyer node recursion (Sec. 3).
//
// Representation (product path; independent of the CPU oracle): a continuous
// PWL function of the share holding y is a sorted vertex list
//     v[i] = (x_i, f_i, s_i),  i = 0..n-1,  n >= 1,
// where f_i = f(x_i) and s_i is the slope on (x_i, x_{i+1}) (s_{n-1} is the
// right tail), plus the left-tail slope sl on (-inf, x_0).  A line is a single
// anchor vertex with s_0 == sl.  Slopes are carried EXACTLY: every slope is a
// copy of a lattice value -(1 +- k) S_{t,j} r^-t created once (as a quote or a
// tail) and never recomputed, so "same slope" is a bitwise test and no
// difference quotient is ever taken.
//
// All functions are stored DISCOUNTED to time 0: zh_t = z_t / r^t.  Then the
// paper's "w_t / r" disappears: wh_t = max(zh_{t+1}^u, zh_{t+1}^d)
// = (w_t / r) / r^t, and the slope restriction to [-S^a_t, -S^b_t] becomes a
// restriction to [-S^a_t r^-t, -S^b_t r^-t] (restriction commutes with
// positive scaling).  At t = 0, r^0 = 1, so prices read off unchanged.
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define AMTC_HD __host__ __device__ __forceinline__
#else
#define AMTC_HD inline
#endif

namespace amtc {

struct Vtx {
    double x, f, s;
};

// status bits raised by the device algebra
enum : int { DEV_OK = 0, DEV_OVERFLOW = 1, DEV_UNBOUNDED = 2 };

// Rounding guards (reading R10: they change values by rounding-level amounts
// only and keep the representation free of rounding-made micro-pieces):
//  * two values closer than TOL_F (|a| + |b| + 1) are "equal": a function does
//    not "cross" another it merely touches (ties are broken by slope);
//  * a piece shorter than TOL_X (1 + |x|) is folded into its neighbour.
constexpr double TOL_F = 1e-14;
constexpr double TOL_X = 1e-12;
AMTC_HD double ftol(double a, double b) { return TOL_F * (fabs(a) + fabs(b) + 1.0); }
AMTC_HD double xtol(double x) { return TOL_X * (1.0 + fabs(x)); }

// Forward emitter: appends vertices in increasing x, skipping non-kinks
// (same slope as the previous piece) and folding zero-length pieces.
struct Emit {
    Vtx* out;
    int m, cap;
    int stride;     // element stride of `out` (1 = contiguous; 32 = lane-interleaved slots)
    double sl;      // left-tail slope of the function being built
    double last_s;  // slope of the last piece emitted (sl if none)
    double ax, af;  // anchor candidate (first point offered)
    bool has_anchor;
    int err;

    AMTC_HD void init(Vtx* o, int c, double left_slope, int str = 1) {
        out = o; m = 0; cap = c; stride = str; sl = left_slope; last_s = left_slope; has_anchor = false;
        err = DEV_OK;
    }
    AMTC_HD Vtx& at(int i) { return out[i * stride]; }
    AMTC_HD void push(double x, double f, double s) {
        if (!has_anchor) { ax = x; af = f; has_anchor = true; }
        if (s == last_s) return;  // not a kink
        if (m > 0 && !(x > at(m - 1).x + xtol(x))) {
            // (near) zero-length piece (coincident or rounding-made vertex):
            // the previous vertex turns directly into slope s
            at(m - 1).s = s;
            double left = (m > 1) ? at(m - 2).s : sl;
            if (left == s) m--;  // the previous vertex is no longer a kink
            last_s = s;
            return;
        }
        if (m >= cap) { err |= DEV_OVERFLOW; return; }
        Vtx& o = at(m);
        o.x = x; o.f = f; o.s = s;
        m++;
        last_s = s;
    }
    // close the function: a line keeps one anchor vertex
    AMTC_HD int finish() {
        if (m == 0) {
            if (cap < 1) { err |= DEV_OVERFLOW; return 0; }
            at(0).x = has_anchor ? ax : 0.0;
            at(0).f = has_anchor ? af : 0.0;
            at(0).s = sl;
            m = 1;
        }
        return m;
    }
};

// A read-only function view.
struct Fn {
    const Vtx* p;
    int n;
    double sl;
    int stride;  // element stride of p (1 = contiguous; 32 = lane-interleaved slots)
    AMTC_HD const Vtx& v(int i) const { return p[i * stride]; }
    AMTC_HD double slope_right(int i) const { return i < 0 ? sl : v(i).s; }
};
AMTC_HD Fn make_fn(const Vtx* p, int n, double sl, int stride = 1) {
    Fn F;
    F.p = p; F.n = n; F.sl = sl; F.stride = stride;
    return F;
}

// value at y of the piece that starts at vertex i (i = -1: the left tail,
// anchored at vertex 0)
AMTC_HD double piece_at(const Fn& F, int i, double y) {
    const Vtx& a = F.v(i < 0 ? 0 : i);
    double s = i < 0 ? F.sl : a.s;
    return fma(s, y - a.x, a.f);
}

// Pointwise max (is_max) or min of F and G (P:118 w = max(z^u, z^d)
// z = max(u, v); P:142 z = min(u, v)).  A two-pointer sweep over the union of
// both vertex sets; between consecutive events both are affine, so at most one
// crossing per interval (and per tail).
AMTC_HD int envelope(const Fn& F, const Fn& G, bool is_max, Emit& E) {
    // winner on the left tail
    double xe0 = fmin(F.v(0).x, G.v(0).x);
    double eF0 = piece_at(F, -1, xe0), eG0 = piece_at(G, -1, xe0);
    bool curF;
    if (F.sl != G.sl) curF = is_max ? (F.sl < G.sl) : (F.sl > G.sl);
    else curF = is_max ? (eF0 >= eG0) : (eF0 <= eG0);
    // a left-tail winner that is only tied at the first event does not cross
    E.init(E.out, E.cap, curF ? F.sl : G.sl, E.stride);
    int iF = -1, iG = -1;
    double sF = F.sl, sG = G.sl;
    double xprev = -INFINITY;
    double eF = eF0, eG = eG0, xe = xe0;
    while (iF + 1 < F.n || iG + 1 < G.n) {
        double xF = (iF + 1 < F.n) ? F.v(iF + 1).x : INFINITY;
        double xG = (iG + 1 < G.n) ? G.v(iG + 1).x : INFINITY;
        xe = fmin(xF, xG);
        eF = (xF == xe) ? F.v(iF + 1).f : piece_at(F, iF, xe);
        eG = (xG == xe) ? G.v(iG + 1).f : piece_at(G, iG, xe);
        // crossing inside (xprev, xe): the current winner lost strictly at xe
        const double tl = ftol(eF, eG);
        bool lost = curF ? (is_max ? (eG > eF + tl) : (eG < eF - tl)) : (is_max ? (eF > eG + tl) : (eF < eG - tl));
        if (lost) {
            // sF == sG only if rounding flipped the order of parallel lines
            double yc = (sF != sG) ? xe - (eF - eG) / (sF - sG) : xe;
            yc = fmin(fmax(yc, xprev), xe);
            curF = !curF;
            double fc = curF ? piece_at(F, iF, yc) : piece_at(G, iG, yc);
            E.push(yc, fc, curF ? sF : sG);
        }
        if (xF == xe) { iF++; sF = F.v(iF).s; }
        if (xG == xe) { iG++; sG = G.v(iG).s; }
        if (fabs(eF - eG) > tl) curF = is_max ? (eF > eG) : (eF < eG);
        else curF = is_max ? (sF >= sG) : (sF <= sG);  // tie: the one that wins to the right
        E.push(xe, is_max ? fmax(eF, eG) : fmin(eF, eG), curF ? sF : sG);
        xprev = xe;
    }
    // right tails: the loser may overtake
    {
        double sw = curF ? sF : sG, sLo = curF ? sG : sF;
        double fw = curF ? eF : eG, fLo = curF ? eG : eF;
        bool overtakes = is_max ? (sLo > sw) : (sLo < sw);
        if (overtakes) {
            double yc = xe + (fw - fLo) / (sLo - sw);
            if (!(yc >= xe)) yc = xe;
            double fc = fma(sLo, yc - xe, fLo);
            E.push(yc, fc, sLo);
        }
    }
    return E.finish();
}

// Reverse emitter for the right-to-left restriction pass: writes vertices at
// decreasing addresses out[cap-1], out[cap-2], ...  The caller only offers
// true kinks (it knows both neighbouring slopes).
struct EmitRev {
    Vtx* out;
    int m, cap, stride;
    int err;
    AMTC_HD void init(Vtx* o, int c, int str = 1) { out = o; m = 0; cap = c; stride = str; err = DEV_OK; }
    AMTC_HD Vtx& at(int i) { return out[i * stride]; }
    AMTC_HD void push(double x, double f, double s_right) {
        if (m > 0) {
            Vtx& last = at(cap - m);  // the vertex to the right
            if (!(x < last.x - xtol(x))) {  // (near) zero-length piece: fold into the right vertex
                return;
            }
        }
        if (m >= cap) { err |= DEV_OVERFLOW; return; }
        Vtx& o = at(cap - 1 - m);
        o.x = x; o.f = f; o.s = s_right;
        m++;
    }
};

// Slope restriction ("restricted within the interval [-S^a_t, -S^b_t]")
// of a possibly non-convex W to [lo, hi], as the infimal convolution with the
// rebalancing cost (buy at -lo, sell at -hi), computed in two monotone passes:
//   pass A (right to left):  A(y) = inf_{y' >= y} W(y') + lo (y - y')
//   pass B (left to right):  V(y) = inf_{y' <= y} A(y') + hi (y - y')
// (sell-then-buy is never cheaper than a direct trade, so V = min of the buy
// and sell branches, reading R7).  Each pass keeps A = W ("tracking") or a
// line of slope lo / hi ("flat"), switching at vertices or single crossings.
//
// Pass A writes A reversed into `abuf` (cap entries, the last nA used).
AMTC_HD int restrict_pass_a(const Fn& W, double lo, Vtx* abuf, int cap, int& nA,
                                               double& slA, int stride = 1) {
    EmitRev R;
    R.init(abuf, cap, stride);
    if (W.v(W.n - 1).s < lo) { nA = 0; return DEV_UNBOUNDED; }
    bool flat = false;
    double Lx = 0.0, Lf = 0.0;
    double cur_s = W.v(W.n - 1).s;  // A's slope just right of the current vertex
    for (int i = W.n - 1; i >= 0; --i) {
        double x = W.v(i).x, fw = W.v(i).f;
        double sp = (i > 0) ? W.v(i - 1).s : W.sl;  // slope of the piece left of x
        double Ax, s_left;
        bool cross = false;
        double yc = 0.0, fc = 0.0;
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
                double d = fw - Ax;
                if (d <= ftol(fw, Ax)) {  // W touches the flat line at x: track from here
                    flat = false; Ax = fw; s_left = sp;
                } else {
                    yc = x - d / (sp - lo);
                    if (i == 0 || yc > W.v(i - 1).x) {
                        cross = true;
                        fc = fma(lo, yc - Lx, Lf);
                    }
                }
            }
        }
        if (s_left != cur_s) R.push(x, Ax, cur_s);
        cur_s = s_left;
        if (cross) {
            R.push(yc, fc, lo);
            flat = false;
            cur_s = sp;
        }
    }
    slA = cur_s;
    if (R.m == 0) {  // a line: anchor at the last vertex
        R.push(W.v(0).x, flat ? fma(lo, W.v(0).x - Lx, Lf) : W.v(0).f, cur_s);
    }
    nA = R.m;
    return R.err;
}

// Pass B over A (forward), emitting V through E (whose left slope is A's).
AMTC_HD int restrict_pass_b(const Fn& A, double hi, Emit& E) {
    if (A.sl > hi) return DEV_UNBOUNDED;
    E.init(E.out, E.cap, A.sl, E.stride);
    bool flat = false;
    double Mx = 0.0, Mf = 0.0;
    for (int i = 0; i < A.n; ++i) {
        double x = A.v(i).x, fa = A.v(i).f, sp = A.v(i).s;  // piece right of x
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
                double d = fa - Bx;
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
        E.push(x, Bx, s_right);
        if (cross) {
            E.push(yc, fc, sp);
            flat = false;
        }
    }
    E.finish();
    return E.err;
}

}  // namespace amtc

namespace amtc {

// One node of the seller (party 0) or buyer (party 1)
// recursion on discounted functions.  U, D: the children z_{t+1,j},
// z_{t+1,j+1}; [lo, hi] = [-S^a_t, -S^b_t] r^-t; (ux, uf): the vertex of the
// discounted exercise function u_t (seller: (zeta, xi r^-t), buyer:
// (-zeta, -xi r^-t)) whose tails are lo and hi.
// Scratch: r0 and r1, b vertices each.  The result Z is left in r1[0..nZ).
AMTC_HD int node_update(const Fn& U, const Fn& D, double lo, double hi, double ux, double uf, bool seller,
                        Vtx* r0, Vtx* r1, int b, int& nZ, double& slZ, int stride = 1) {
    // w = max(z^u, z^d)  (discounted, so no division by r)
    Emit E;
    E.out = r0;
    E.cap = b;
    E.stride = stride;
    envelope(U, D, true, E);
    int err = E.err;
    if (err) return err;
    const Fn W = make_fn(r0, E.m, E.sl, stride);
    // v = restriction of w to [lo, hi]  (reading R7)
    int nA;
    double slA;
    err |= restrict_pass_a(W, lo, r1, b, nA, slA, stride);
    if (err) return err;
    const Fn Af = make_fn(r1 + (size_t)(b - nA) * stride, nA, slA, stride);
    Emit EV;
    EV.out = r0;
    EV.cap = b;
    EV.stride = stride;
    err |= restrict_pass_b(Af, hi, EV);
    if (err) return err;
    const Fn Vf = make_fn(r0, EV.m, EV.sl, stride);
    // z = max(u, v) seller / min(u, v) buyer
    Vtx uv;
    uv.x = ux;
    uv.f = uf;
    uv.s = hi;
    const Fn Uf = make_fn(&uv, 1, lo, 1);
    Emit EZ;
    EZ.out = r1;
    EZ.cap = b;
    EZ.stride = stride;
    envelope(Uf, Vf, seller, EZ);
    nZ = EZ.m;
    slZ = EZ.sl;
    return EZ.err;
}

}  // namespace amtc
