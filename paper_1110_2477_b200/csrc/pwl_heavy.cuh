// pwl_heavy.cuh -- warp-cooperative node update for HEAVY node functions (the
// buyer's "sawtooth" of calls / bull spreads: thousands of vertices, DESIGN.md
// section 5).  Three implementations of the same data-parallel form:
//   node_update_block  (default, tier 3) block-synchronous: merged events in
//                      blocks of 32 from shared merge windows (ranks by binary
//                      search in shared memory), W compacted to scratch, then
//                      per-W-vertex emission of z; no dependent global loads.
//   node_update        (fallback for rare shapes) lane-contiguous: lane i runs
//                      the sequential generator over 1/32 of the events.
//   node_update_chunk  (fallback of the fallback) chunk-synchronous with merge-
//                      path binary searches in global memory.
//
// Data-parallel form of one node (Sec. 3; reading A7): with
//   W = max(U, D)                              (discounted, so no /r)
//   g_j = W_j - lo x_j,  h_j = W_j - hi x_j    over the vertices x_j of W,
//   M_j = min_{i >= j} g_i,  P_j = min_{i <= j} h_i,
// the restriction of W to slopes [lo, hi] is, on the piece (x_j, x_{j+1}),
//   v(y) = min( W(y), lo y + M_{j+1}, hi y + P_j )
// (the infimum of a piecewise-linear function over a half line is attained at
// its end point or at a vertex; the tails are monotone when d < r < u), and
// z = max(u, v) (seller) / min(u, v) (buyer).  The vertex owner
// of piece j emits z's vertices on [x_j, x_{j+1}); vertices are staged per lane,
// de-duplicated against the slope arriving from the left, folded when closer
// than xtol (reading A10) and compacted with a warp prefix sum.
#pragma once
#include "pwl_device.cuh"

namespace amtc {
namespace heavy {

constexpr unsigned FULLM = 0xffffffffu;
constexpr int STAGE = 40;  // staged output vertices per lane per block
constexpr int DEV_FALLBACK = 8;  // node_update_block: use node_update for this node

// merged event k: the k-th vertex of U and D by x (U first on ties)
struct Ev {
    double x, eU, eD, sUL, sUR, sDL, sDR;
    bool skip;  // a D vertex at the x of the previous (U) event, which handled both
};

// number of U events among the first k (merge path), searched in [lo, hi]
__device__ __forceinline__ int split(const Fn& U, const Fn& D, int k, int lo, int hi) {
    lo = max(lo, k - D.n);
    hi = min(hi, min(k, U.n));
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (U.v(mid).x <= D.v(k - mid - 1).x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ Ev event_at(const Fn& U, const Fn& D, int k, int a) {
    Ev e;
    e.skip = false;
    const int b = k - a;
    const bool isU = a < U.n && (b >= D.n || U.v(a).x <= D.v(b).x);
    if (isU) {
        const Vtx u = U.v(a);
        e.x = u.x; e.eU = u.f; e.sUR = u.s; e.sUL = a > 0 ? U.v(a - 1).s : U.sl;
        if (b < D.n && D.v(b).x == e.x) {  // coincident vertices: one event
            const Vtx d = D.v(b);
            e.eD = d.f; e.sDR = d.s; e.sDL = b > 0 ? D.v(b - 1).s : D.sl;
        } else {
            const int p = b - 1;
            const Vtx d = D.v(p < 0 ? 0 : p);
            const double s = p < 0 ? D.sl : d.s;
            e.eD = fma(s, e.x - d.x, d.f); e.sDL = s; e.sDR = s;
        }
    } else {
        const Vtx d = D.v(b);
        e.x = d.x; e.eD = d.f; e.sDR = d.s; e.sDL = b > 0 ? D.v(b - 1).s : D.sl;
        if (a > 0 && U.v(a - 1).x == e.x) {
            e.skip = true;
            const Vtx u = U.v(a - 1);
            e.eU = u.f; e.sUR = u.s; e.sUL = a > 1 ? U.v(a - 2).s : U.sl;
        } else {
            const int p = a - 1;
            const Vtx u = U.v(p < 0 ? 0 : p);
            const double s = p < 0 ? U.sl : u.s;
            e.eU = fma(s, e.x - u.x, u.f); e.sUL = s; e.sUR = s;
        }
    }
    return e;
}

// winner of max(U, D) just right / just left of the event (ties: by slope)
__device__ __forceinline__ bool winR(const Ev& e) {
    const double tl = ftol(e.eU, e.eD);
    return fabs(e.eU - e.eD) > tl ? e.eU > e.eD : e.sUR >= e.sDR;
}
__device__ __forceinline__ bool winL(const Ev& e) {
    const double tl = ftol(e.eU, e.eD);
    return fabs(e.eU - e.eD) > tl ? e.eU > e.eD : e.sUL <= e.sDL;
}

// one vertex of W: position, value, slopes left / right
struct WV {
    double x, f, sL, sR;
};

// the (up to 3) vertices of W owned by one event, in x order
struct WV3 {
    WV v0, v1, v2;
    int n;
    __device__ __forceinline__ WV get(int q) const { return q == 0 ? v0 : (q == 1 ? v1 : v2); }
};

// W's vertices produced by event e: a crossing on (x_prev, x), the vertex at
// x, and (last event only) a crossing on the right tail.  wRp: winner just
// right of the previous event (for the first event: the left-tail winner);
// wInf: the right-tail winner.
__device__ __forceinline__ WV3 w_vertices(const Ev& e, bool valid, double x_prev, bool wRp, bool last,
                                          bool wInf) {
    WV3 r;
    r.n = 0;
    if (!valid || e.skip) return r;
    const bool wl = winL(e), wr = winR(e);
    WV c0, c1, c2;
    bool h0 = false, h1 = false, h2 = false;
    if (wRp != wl) {  // crossing on (x_prev, x)
        const double e_w = wl ? e.eU : e.eD, e_o = wl ? e.eD : e.eU;
        const double s_w = wl ? e.sUL : e.sDL, s_o = wl ? e.sDL : e.sUL;
        if (s_w != s_o) {
            const double y = e.x - (e_w - e_o) / (s_w - s_o);
            if (y > x_prev && y < e.x) {
                c0 = WV{y, fma(s_w, y - e.x, e_w), s_o, s_w};
                h0 = true;
            }
        }
    }
    const double sWL = wl ? e.sUL : e.sDL, sWR = wr ? e.sUR : e.sDR;
    if (sWL != sWR) {
        c1 = WV{e.x, fmax(e.eU, e.eD), sWL, sWR};
        h1 = true;
    }
    if (last && wr != wInf) {  // crossing on (x, +inf)
        const double e_w = wr ? e.eU : e.eD, e_o = wr ? e.eD : e.eU;
        const double s_w = wr ? e.sUR : e.sDR, s_o = wr ? e.sDR : e.sUR;
        if (s_o != s_w) {
            const double y = e.x + (e_w - e_o) / (s_o - s_w);
            if (y > e.x) {
                c2 = WV{y, fma(s_w, y - e.x, e_w), s_w, s_o};
                h2 = true;
            }
        }
    }
    r.v0 = h0 ? c0 : (h1 ? c1 : c2);
    r.v1 = (h0 && h1) ? c1 : c2;
    r.v2 = c2;
    r.n = (int)h0 + (int)h1 + (int)h2;
    return r;
}

// W vertices of the 32 events of block `blk` (lane i: event 32 blk + i)
struct BlockW {
    WV3 w;
    bool valid;
};

struct HCtx {
    Fn U, D;
    int nE;
    int klast;     // the last event that is not a skip (it owns the right-tail crossing)
    bool tailL_U;  // winner at -inf is U
    bool wInf_U;   // winner at +inf is U
};

__device__ __forceinline__ HCtx make_ctx(const Fn& U, const Fn& D) {
    HCtx h;
    h.U = U;
    h.D = D;
    h.nE = U.n + D.n;
    // coincident last vertices: the last event (D's) is a skip handled by U's
    h.klast = (U.v(U.n - 1).x == D.v(D.n - 1).x) ? h.nE - 2 : h.nE - 1;
    const double sUr = U.v(U.n - 1).s, sDr = D.v(D.n - 1).s;
    // ties (parallel tails): decided by the value far out, i.e. at the outermost vertex
    if (U.sl != D.sl) h.tailL_U = U.sl < D.sl;
    else {
        const double x0 = fmin(U.v(0).x, D.v(0).x);
        h.tailL_U = piece_at(U, -1, x0) >= piece_at(D, -1, x0);
    }
    if (sUr != sDr) h.wInf_U = sUr > sDr;
    else {
        const double x1 = fmax(U.v(U.n - 1).x, D.v(D.n - 1).x);
        h.wInf_U = piece_at(U, U.n - 1, x1) >= piece_at(D, D.n - 1, x1);
    }
    return h;
}

__device__ __forceinline__ BlockW block_w(const HCtx& h, int blk, int lane) {
    const int k0 = blk * 32;
    const int a0 = split(h.U, h.D, k0, 0, h.U.n);
    const int k = k0 + lane;
    BlockW B;
    B.valid = k < h.nE;
    const int kk = B.valid ? k : h.nE - 1;
    const int a = split(h.U, h.D, kk, a0, a0 + lane);
    const Ev e = event_at(h.U, h.D, kk, a);
    const bool wr = winR(e);
    double x_prev = __shfl_up_sync(FULLM, e.x, 1);
    bool wRp = __shfl_up_sync(FULLM, (int)wr, 1) != 0;
    if (lane == 0) {
        if (k0 == 0) {
            x_prev = -INFINITY;
            wRp = h.tailL_U;
        } else {
            const int ap = split(h.U, h.D, k0 - 1, max(a0 - 1, 0), a0);
            const Ev ep = event_at(h.U, h.D, k0 - 1, ap);
            x_prev = ep.x;
            wRp = winR(ep);
        }
    }
    B.w = w_vertices(e, B.valid, x_prev, wRp, k == h.klast, h.wInf_U);
    return B;
}

// ---------------------------------------------------------------------------
// z = OP(u, v) on a piece, v = min(W line, lo y + M, hi y + P)
// ---------------------------------------------------------------------------
struct Line {
    double x0, f0, s;
    __device__ __forceinline__ double at(double y) const { return fma(s, y - x0, f0); }
};

struct PCtx {
    double lo, hi, ux, uf;
    bool seller;
};

// z's state just right (right = true) or just left of the finite position y:
// returns z's slope; vi = active v line (0 W, 1 M, 2 P), zU = u wins, zval = z(y)
__device__ __forceinline__ double z_side(const Line& LW, const Line& LM, bool hasM, const Line& LP, bool hasP,
                                         const PCtx& c, double y, bool right, int& vi, bool& zU, double& zval) {
    vi = 0;
    double vv = LW.at(y), vs = LW.s;
    if (hasM) {
        const double m = LM.at(y);
        const double tl = ftol(m, vv);
        if (m < vv - tl || (fabs(m - vv) <= tl && (right ? LM.s < vs : LM.s > vs))) { vi = 1; vv = m; vs = LM.s; }
    }
    if (hasP) {
        const double p = LP.at(y);
        const double tl = ftol(p, vv);
        if (p < vv - tl || (fabs(p - vv) <= tl && (right ? LP.s < vs : LP.s > vs))) { vi = 2; vv = p; vs = LP.s; }
    }
    const double us = (right ? (y >= c.ux) : (y > c.ux)) ? c.hi : c.lo;
    const double uv = fma(us, y - c.ux, c.uf);
    const double tl = ftol(uv, vv);
    bool uw;
    if (fabs(uv - vv) > tl) uw = c.seller ? (uv > vv) : (uv < vv);
    else uw = c.seller ? (right ? us > vs : us < vs) : (right ? us < vs : us > vs);
    zU = uw;
    zval = c.seller ? fmax(uv, vv) : fmin(uv, vv);
    return uw ? us : vs;
}

// where line A meets line B, from values at the finite reference point ref
__device__ __forceinline__ double cross_at(const Line& A, const Line& B, double ref) {
    return ref - (A.at(ref) - B.at(ref)) / (A.s - B.s);
}

// the crossing y of A with B (A.s < B.s: A comes from above; rising = true:
// A.s > B.s, A comes from below) replaces nx if p_in < y < nx.  In exact
// arithmetic y < nx iff A is already past B at a finite nx.
__device__ __forceinline__ void try_cross(const Line& A, const Line& B, double ref, double p_in, double& nx,
                                          bool rising) {
    if (isfinite(nx)) {
        const double a = A.at(nx), b = B.at(nx);
        if (rising ? !(a > b) : !(a < b)) return;
    }
    const double y = cross_at(A, B, ref);
    if (y > p_in && y < nx) nx = y;
}

// per-lane staging of output vertices (global scratch, lane-interleaved)
struct Stage {
    Vtx* buf;   // STAGE x 32 (global, lane-interleaved)
    Vtx* sbuf;  // optional: rows 0 and 1 in shared memory (nullptr: all rows in buf)
    int lane, m, err;
    double last_s;  // slope after the last staged vertex
    __device__ __forceinline__ Vtx& at(int q) const {
        return (q < 2 && sbuf) ? sbuf[q * 32 + lane] : buf[q * 32 + lane];
    }
    __device__ __forceinline__ void push(double x, double f, double s) {
        if (m > 0) {
            Vtx& p = at(m - 1);
            if (!(x > p.x + xtol(x))) {
                // (near) zero-length piece: the previous vertex turns into slope s
                // directly (reading A10, as pwl_device.cuh's Emit)
                p.s = s;
                if (m > 1 && at(m - 2).s == s) m--;  // no longer a kink
                last_s = s;
                return;
            }
        }
        if (m >= STAGE) { err |= DEV_OVERFLOW; return; }
        Vtx& o = at(m);
        o.x = x; o.f = f; o.s = s;
        m++;
        last_s = s;
    }
};

// Stage z's vertices strictly inside (a, b); a finite or -inf (then the state
// at -inf is given: v = the M line, u = its lo line, zU0 = u wins there).
// s_cur: z's slope just right of a.  Returns z's slope just left of b.
// vi0 >= 0: z's state just right of a is already known (vi0, zU0: z_side's
// outputs at a), otherwise it is evaluated here.
// ENTRY_KNOWN: the caller guarantees vi0 >= 0 or a = -inf, so the entry never
// evaluates z_side (one inlined copy less in the block update's sweep C).
template <class Out, bool ENTRY_KNOWN = false>
__device__ __forceinline__ double emit_open(double a, double b, const Line& LW, const Line& LM, bool hasM,
                                            const Line& LP, bool hasP, const PCtx& c, double s_cur, bool zU0,
                                            Out& st, int vi0 = -1) {
    double pos = a;
    int vi;
    bool zU;
    double zv;
    if (vi0 >= 0) { vi = vi0; zU = zU0; }
    else if (!ENTRY_KNOWN && isfinite(a)) z_side(LW, LM, hasM, LP, hasP, c, a, true, vi, zU, zv);
    else { vi = hasM ? 1 : 0; zU = zU0; }
    // events closer than xtol() to either end are rounding images of the end
    // vertex itself (e.g. the M line passes through the vertex that defines it)
    const double b_in = isfinite(b) ? b - xtol(b) : b;
    for (int it = 0; it < 10; ++it) {
        const Line V = vi == 0 ? LW : (vi == 1 ? LM : LP);
        const double ref = isfinite(pos) ? pos : c.ux;
        const double p_in = isfinite(pos) ? pos + xtol(pos) : pos;
        const double us = (pos >= c.ux) ? c.hi : c.lo;
        const Line Uq{c.ux, c.uf, us};
        double nx = b_in;
        // v switches to a line with a smaller slope that comes from above
        // (each crossing is first screened by the sign of the difference at nx,
        // so the division runs only for a crossing that can still win)
#ifdef AMTC_ROLLED_CROSS
        // the same four candidates in the same order through ONE inlined copy of
        // try_cross (code size: sweep C is instruction-fetch bound)
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            Line A, Bq;
            bool on, rising = false;
            if (k < 3) {
                A = k == 0 ? LM : (k == 1 ? LP : LW);
                Bq = V;
                on = (k == 0 ? (vi != 1 && hasM) : (k == 1 ? (vi != 2 && hasP) : (vi != 0))) && A.s < V.s;
            } else {
                if (pos < c.ux && c.ux < nx) nx = c.ux;  // u's kink
                A = zU ? V : Uq;                         // z's loser overtakes the winner
                Bq = zU ? Uq : V;
                rising = c.seller;
                on = c.seller ? (A.s > Bq.s) : (A.s < Bq.s);
            }
            if (on) try_cross(A, Bq, ref, p_in, nx, rising);
        }
#else
        if (vi != 1 && hasM && LM.s < V.s) try_cross(LM, V, ref, p_in, nx, false);
        if (vi != 2 && hasP && LP.s < V.s) try_cross(LP, V, ref, p_in, nx, false);
        if (vi != 0 && LW.s < V.s) try_cross(LW, V, ref, p_in, nx, false);
        // u's kink
        if (pos < c.ux && c.ux < nx) nx = c.ux;
        // z's loser overtakes the winner
        {
            const Line& Wn = zU ? Uq : V;
            const Line& Ls = zU ? V : Uq;
            if (c.seller ? (Ls.s > Wn.s) : (Ls.s < Wn.s)) try_cross(Ls, Wn, ref, p_in, nx, c.seller);
        }
#endif
        if (!(nx < b_in)) break;
        pos = nx;
        const double s_new = z_side(LW, LM, hasM, LP, hasP, c, pos, true, vi, zU, zv);
        if (s_new != s_cur) {
            st.push(pos, zv, s_new);
            s_cur = s_new;
        }
    }
    return s_cur;
}

// z = W on the whole piece [x, xn) of the W vertex (x, f, s) (the common case
// inside the buyer's sawtooth): v = W there -- the piece's slope lies in
// [lo, hi], the M line (slope lo <= s) starts above W by more than ftol (or
// within ftol when parallel to the piece) and does not dip below W before xn, the P line (slope hi >= s) starts at or above
// W within ftol -- and u loses to v by more than ftol at the piece's ends and
// at u's kink inside it.  Then the piece emits just its vertex (x, f, s),
// which is what z_side + emit_open produce in that case, without their
// per-line crossing searches.
__device__ __forceinline__ bool piece_is_w(double x, double f, double s, double xn, double Mnext, double Pj,
                                           const PCtx& c) {
    if (!(s >= c.lo && s <= c.hi)) return false;
    const double p = fma(c.hi, x, Pj);
    if (p < f - ftol(p, f)) return false;
    const bool fin = isfinite(xn);
    const double wn = fin ? fma(s, xn - x, f) : 0.0;
    if (isfinite(Mnext)) {
        if (!fin) return false;
        const double m = fma(c.lo, x, Mnext);
        const double tm = ftol(m, f);
        // a tie at x keeps W only when the M line is parallel to the piece (z_side's slope rule)
        if (!(m > f + tm || (s == c.lo && m >= f - tm))) return false;
        const double mn = fma(c.lo, xn, Mnext);
        if (mn < wn - ftol(mn, wn)) return false;
    }
    const double u0 = fma(x >= c.ux ? c.hi : c.lo, x - c.ux, c.uf);
    if (c.seller) {
        if (!fin || !(f > u0 + ftol(u0, f))) return false;
        const double un = fma(xn > c.ux ? c.hi : c.lo, xn - c.ux, c.uf);
        return wn > un + ftol(un, wn);
    }
    if (!(u0 > f + ftol(u0, f))) return false;
    if (fin) {
        const double un = fma(xn > c.ux ? c.hi : c.lo, xn - c.ux, c.uf);
        if (!(un > wn + ftol(un, wn))) return false;
    }
    if (x < c.ux && c.ux < xn) {
        const double wk = fma(s, c.ux - x, f);
        if (!(c.uf > wk + ftol(c.uf, wk))) return false;
    }
    return true;
}

#ifndef AMTC_HEAVY_STAT
#define AMTC_HEAVY_STAT(i)
#endif

// Code size: the block update is instruction-fetch bound (DESIGN.md section 8:
// half of the kernel's stall samples are no_inst), so the 5-step warp scans and
// the window binary searches are rolled loops (config 4: 8.88 -> 7.90 s/step for
// the scans alone) and sweep C's emit_open calls never inline the entry z_side.
// -DAMTC_UNROLLED_SCANS / -DAMTC_UNROLLED_RANK / -DAMTC_NO_ENTRY_KNOWN restore
// the previous forms for A/B builds.
#ifndef AMTC_NO_ENTRY_KNOWN
#define AMTC_ENTRY_KNOWN_V true
#else
#define AMTC_ENTRY_KNOWN_V false
#endif
// RL (rolled loops) is a template parameter of the scans, the rank searches and
// node_update_block: the 20-warp batch kernel is fetch bound and takes the
// rolled forms; the 16-warp split-mode kernel runs one strip pipeline per tree,
// is bound by the latency of a single warp's update and keeps the unrolled
// forms (config 3: 1.70 s unrolled vs 2.00 s rolled).
#ifndef AMTC_UNROLLED_SCANS
constexpr bool RL_DEFAULT = true;
#else
constexpr bool RL_DEFAULT = false;
#endif

// warp-level scans
template <bool RL = RL_DEFAULT>
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll(RL ? 1 : 5)
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULLM, v, o));
    return v;
}
// exclusive suffix min over lanes > lane
template <bool RL = RL_DEFAULT>
__device__ __forceinline__ double excl_suffix_min(double v, int lane) {
    double x = v;
#pragma unroll(RL ? 1 : 5)
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_down_sync(FULLM, x, o);
        if (lane + o < 32) x = fmin(x, y);
    }
    const double nx = __shfl_down_sync(FULLM, x, 1);
    return lane < 31 ? nx : INFINITY;
}
// exclusive prefix min over lanes < lane
template <bool RL = RL_DEFAULT>
__device__ __forceinline__ double excl_prefix_min(double v, int lane) {
    double x = v;
#pragma unroll(RL ? 1 : 5)
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULLM, x, o);
        if (lane >= o) x = fmin(x, y);
    }
    const double px = __shfl_up_sync(FULLM, x, 1);
    return lane > 0 ? px : INFINITY;
}
// exclusive prefix sum of small non-negative counts (v < 2^B) by bit planes:
// B independent ballots instead of a 5-deep shuffle chain
template <int B>
__device__ __forceinline__ int excl_prefix_sum_bits(int v, int lane, int& total) {
    const unsigned lt = (1u << lane) - 1u;
    int off = 0, tot = 0;
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const unsigned m = __ballot_sync(FULLM, (v >> b) & 1);
        off += __popc(m & lt) << b;
        tot += __popc(m) << b;
    }
    total = tot;
    return off;
}
__device__ __forceinline__ int excl_prefix_sum(int v, int lane, int& total) {
    int x = v;
#pragma unroll(RL_DEFAULT ? 1 : 5)
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLM, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(FULLM, x, 31);
    return x - v;
}

// ---------------------------------------------------------------------------
// the heavy node update
//   scratch: >= 2 * ceil(nE/32) doubles + STAGE * 32 vertices (global, per warp)
//   output:  Z appended to arena at *counter (the caller's bump counter for this
//            arena; only this warp allocates from it meanwhile)
// ---------------------------------------------------------------------------
__device__ __forceinline__ size_t scratch_vertices(int nE) {
    const int nb = (nE + 31) / 32;
    return (size_t)STAGE * 32 + (size_t)(2 * nb * sizeof(double) + sizeof(Vtx) - 1) / sizeof(Vtx) + 1;
}

static __device__ __noinline__ int node_update_chunk(const Fn U, const Fn D, double lo, double hi, double ux, double uf,
                                              bool seller, Vtx* scratch, int scap, Vtx* arena, int* counter,
                                              int acap, int& zoff, int& nZ, int lane) {
    const HCtx h = make_ctx(U, D);
    const int nb = (h.nE + 31) / 32;
    if ((size_t)scap < scratch_vertices(h.nE)) return DEV_OVERFLOW;
    Vtx* stage_buf = scratch;
    double* Mafter = reinterpret_cast<double*>(scratch + STAGE * 32);
    double* Xafter = Mafter + nb;
    // restriction is finite iff W's tails are steeper than the quotes (d < r < u)
    {
        const double sWr = h.wInf_U ? U.v(U.n - 1).s : D.v(D.n - 1).s;
        const double sWl = h.tailL_U ? U.sl : D.sl;
        if (sWr < lo || sWl > hi) return DEV_UNBOUNDED;
    }
    // ---- sweep 1: right to left, suffix minima of g at block boundaries ----
    {
        double Mc = INFINITY, Xc = INFINITY;
        for (int blk = nb - 1; blk >= 0; --blk) {
            const BlockW B = block_w(h, blk, lane);
            double gm = INFINITY, fx = INFINITY;
            for (int q = 0; q < B.w.n; ++q) {
                const WV w = B.w.get(q);
                gm = fmin(gm, fma(-lo, w.x, w.f));
                fx = fmin(fx, w.x);
            }
            if (lane == 0) {
                Mafter[blk] = Mc;
                Xafter[blk] = Xc;
            }
            Mc = fmin(Mc, warp_min(gm));
            Xc = fmin(Xc, warp_min(fx));
        }
    }
    __syncwarp();
    // ---- sweep 2: left to right, emit z ----
    const PCtx c{lo, hi, ux, uf, seller};
    const int base = *counter;  // this warp's allocation point in the arena
    int total = 0;
    int err = DEV_OK;
    double Pc = INFINITY;       // prefix min of h over earlier blocks
    double s_in = lo;           // z's slope arriving from the left (z's left tail is lo)
    bool any_before = false;    // a W vertex in an earlier block
    double last_x = -INFINITY;  // the last vertex written (earlier blocks)
    for (int blk = 0; blk < nb; ++blk) {
        const BlockW B = block_w(h, blk, lane);
        const int nw = B.w.n;
        // lane aggregates
        double gl = INFINITY, hl = INFINITY, fx = INFINITY;
        for (int q = 0; q < nw; ++q) {
            const WV w = B.w.get(q);
            gl = fmin(gl, fma(-lo, w.x, w.f));
            hl = fmin(hl, fma(-hi, w.x, w.f));
            fx = fmin(fx, w.x);
        }
        const double Mr = fmin(excl_suffix_min(gl, lane), Mafter[blk]);  // g over lanes > lane and later blocks
        const double Pl = fmin(excl_prefix_min(hl, lane), Pc);           // h over lanes < lane and earlier blocks
        const double Xr = fmin(excl_suffix_min(fx, lane), Xafter[blk]);  // next W vertex after this lane
        int cntb;
        const int before = excl_prefix_sum(nw > 0 ? 1 : 0, lane, cntb);
        const bool first_overall = !any_before && before == 0 && nw > 0;
        // suffix minima for own vertices: M after vertex q
        double Mq2 = Mr, Mq1 = Mr, Mq0 = Mr;  // M_{j+1} for own vertices 2, 1, 0
        {
            if (nw >= 3) Mq1 = fmin(Mr, fma(-lo, B.w.v2.x, B.w.v2.f));
            if (nw >= 2) Mq0 = fmin(nw >= 3 ? Mq1 : Mr, fma(-lo, B.w.v1.x, B.w.v1.f));
            if (nw == 2) Mq1 = Mr;
        }
        Stage st;
        st.buf = stage_buf;
        st.sbuf = nullptr;
        st.lane = lane;
        st.m = 0;
        st.err = DEV_OK;
        st.last_s = NAN;
        double P = Pl;
        double s_run = NAN;    // z's slope just left of the current position (NaN: from the left lane)
        bool pending = false;  // stage slot 0 is a candidate to check against that slope
        for (int q = 0; q < nw; ++q) {
            const WV w = B.w.get(q);
            const double Mnext = q == 0 ? Mq0 : (q == 1 ? Mq1 : Mq2);
            const double Mj = fmin(fma(-lo, w.x, w.f), Mnext);
            const double xn = (q + 1 < nw) ? B.w.get(q + 1).x : Xr;
            if (q == 0 && first_overall) {
                // left-tail piece (-inf, x_0): v = min(W tail, lo y + M_0); far left v is
                // the M line and u its lo line (parallel): the winner is decided by value
                const Line LW{w.x, w.f, w.sL}, LM{0.0, Mj, lo}, LP{0.0, INFINITY, hi};
                const double mv = LM.at(ux);
                const double tl = ftol(mv, uf);
                const bool zU0 = fabs(uf - mv) > tl ? (seller ? uf > mv : uf < mv) : false;
                s_run = emit_open(-INFINITY, w.x, LW, LM, true, LP, false, c, lo, zU0, st);
            }
            // the vertex at x_j: z's slope just right of it
            int vi;
            bool zU;
            double zv;
            const double Pj = fmin(P, fma(-hi, w.x, w.f));
            const Line LWr{w.x, w.f, w.sR}, LMr{0.0, Mnext, lo}, LPr{0.0, Pj, hi};
            const double sr_ = z_side(LWr, LMr, isfinite(Mnext), LPr, true, c, w.x, true, vi, zU, zv);
            if (s_run != s_run) {  // unknown: decided once the left lane's slope is known
                pending = st.m == 0;
                st.push(w.x, zv, sr_);
            } else if (sr_ != s_run) {
                st.push(w.x, zv, sr_);
            }
            s_run = emit_open(w.x, xn, LWr, LMr, isfinite(Mnext), LPr, true, c, sr_, false, st);
            P = Pj;
        }
        const double s_end = s_run;
        // the slope arriving from the left: z's slope at the end of the nearest
        // earlier lane with W vertices (or of the previous block)
        double s_left = s_in;
        {
            int src = nw > 0 ? lane : -1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULLM, src, o);
                if (lane >= o) src = max(src, y);
            }
            int srcp = __shfl_up_sync(FULLM, src, 1);
            if (lane == 0) srcp = -1;
            const double se = __shfl_sync(FULLM, s_end, srcp < 0 ? 0 : srcp);
            if (srcp >= 0) s_left = se;
            const int lastsrc = __shfl_sync(FULLM, src, 31);
            const double se_last = __shfl_sync(FULLM, s_end, lastsrc < 0 ? 0 : lastsrc);
            if (lastsrc >= 0) s_in = se_last;
        }
        // drop the pending candidate when z has no kink there
        const int skip0 = (pending && stage_buf[lane].s == s_left) ? 1 : 0;
        err |= __reduce_or_sync(FULLM, st.err);
        int cnt = st.m - skip0;
        // fold across lanes (as Emit does within one): a first vertex closer than
        // xtol() to the previous kept vertex is merged into it (that vertex takes
        // its slope), so rounding-made micro-pieces never accumulate
        double f0x = 0.0, fs = 0.0, lx = -INFINITY;
        if (cnt > 0) {
            f0x = stage_buf[skip0 * 32 + lane].x;
            fs = stage_buf[skip0 * 32 + lane].s;
            lx = stage_buf[(st.m - 1) * 32 + lane].x;
        }
        int prevl = cnt > 0 ? lane : -1;  // nearest lane <= this one with vertices
        int nextl = cnt > 0 ? lane : 32;  // nearest lane >= this one with vertices
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULLM, prevl, o);
            if (lane >= o) prevl = max(prevl, y);
            const int z = __shfl_down_sync(FULLM, nextl, o);
            if (lane + o < 32) nextl = min(nextl, z);
        }
        int pl = __shfl_up_sync(FULLM, prevl, 1);
        if (lane == 0) pl = -1;
        int nl = __shfl_down_sync(FULLM, nextl, 1);
        if (lane == 31) nl = 32;
        const double px = __shfl_sync(FULLM, lx, pl < 0 ? 0 : pl);
        const double prev_x = pl < 0 ? last_x : px;
        const bool fold = cnt > 0 && !(f0x > prev_x + xtol(f0x));
        const int nfold = __shfl_sync(FULLM, (int)fold, nl > 31 ? 0 : nl);
        const double nfs = __shfl_sync(FULLM, fs, nl > 31 ? 0 : nl);
        if (cnt > 0 && nl <= 31 && nfold) stage_buf[(st.m - 1) * 32 + lane].s = nfs;  // absorb the next lane's first
        if (fold && pl < 0 && total > 0) arena[base + total - 1].s = fs;               // into the previous block
        const int drop_first = (fold && (pl >= 0 || total > 0)) ? 1 : 0;
        cnt -= drop_first;
        int tot;
        const int off = excl_prefix_sum(cnt, lane, tot);
        if (base + total + tot > acap) err |= DEV_OVERFLOW;
        if (err) break;
        for (int q = 0; q < cnt; ++q)
            arena[base + total + off + q] = stage_buf[(q + skip0 + drop_first) * 32 + lane];
        total += tot;
        {
            const int lastl = __shfl_sync(FULLM, prevl, 31);
            const double lxl = __shfl_sync(FULLM, lx, lastl < 0 ? 0 : lastl);
            if (lastl >= 0) last_x = lxl;
        }
        Pc = fmin(Pc, warp_min(hl));
        any_before = any_before || (cntb > 0);
        __syncwarp();
    }
    if (!err && total == 0) {
        // z is a single line (cannot happen for a heavy node; kept for safety)
        if (base + 1 > acap) err |= DEV_OVERFLOW;
        else if (lane == 0) arena[base] = Vtx{0.0, fma(lo, -ux, uf), lo};
        total = 1;
    }
    if (lane == 0 && !err) *counter = base + total;
    __syncwarp();
    zoff = base;
    nZ = total;
    return err;
}


// ===========================================================================
// Lane-contiguous heavy update (the default): lane i runs a sequential,
// forward W generator over its own segment of the merged event sequence
// (carried merge state, as the per-lane node update does), so the per-event
// cost is that of the sequential algorithm; the segments are joined by warp
// scans (suffix minima of g, prefix minima of h, look-ahead to the next W
// vertex, the slope arriving from the left) and a count-then-write pass.
// M_{j+1} = min over later W vertices of g: inside a lane it is g_{j+1} or the
// value at a later local minimum of g (recorded in pass 1; at most LMAX).
// Anything unusual (too many local minima, a fold into a dropped vertex)
// falls back to node_update_chunk.
// ===========================================================================
constexpr int LMAX = 6;

// forward W generator over merged events [k, kend)
struct WGen {
    const Fn* U;
    const Fn* D;
    int k, kend, a;      // next event, end, U events before k
    double x_prev;       // position of the previous event
    bool wRp;            // winner (U?) just right of the previous event
    int klast;
    bool wInf;
    // pending vertices of the current event (up to 3)
    WV3 cur;
    int q;

    __device__ __forceinline__ void init(const HCtx& h, int k0, int k1, int lane_dummy) {
        U = &h.U;
        D = &h.D;
        k = k0;
        kend = k1;
        klast = h.klast;
        wInf = h.wInf_U;
        a = split(h.U, h.D, k0, 0, h.U.n);
        if (k0 == 0) {
            x_prev = -INFINITY;
            wRp = h.tailL_U;
        } else {
            const int ap = split(h.U, h.D, k0 - 1, max(a - 1, 0), a);
            const Ev ep = event_at(h.U, h.D, k0 - 1, ap);
            x_prev = ep.x;
            wRp = winR(ep);
        }
        cur.n = 0;
        q = 0;
        (void)lane_dummy;
    }
    // next W vertex; false at the end of the segment
    __device__ __forceinline__ bool next(WV& w) {
        while (q >= cur.n) {
            if (k >= kend) return false;
            const Ev e = event_at(*U, *D, k, a);
            cur = w_vertices(e, true, x_prev, wRp, k == klast, wInf);
            q = 0;
            // advance the merge position: event k consumed one vertex of U or D
            const int b = k - a;
            const bool isU = a < U->n && (b >= D->n || U->v(a).x <= D->v(b).x);
            a += isU ? 1 : 0;
            x_prev = e.x;
            wRp = winR(e);
            ++k;
        }
        w = cur.get(q++);
        return true;
    }
};

// register emitter: in-lane folding (as Emit) with the previous vertex kept
// in registers; out == nullptr counts only
struct LEmit {
    Vtx* out;
    int m;
    bool have;
    double lx, ls;   // last vertex written: x and slope
    double ps;       // slope before the last vertex (NaN if unknown)
    int err;
    __device__ __forceinline__ void push(double x, double f, double s) {
        if (have && !(x > lx + xtol(x))) {  // (near) zero-length piece
            if (m == 1) err |= 8;  // folded into the first vertex (may be dropped): bail out
            if (out) out[m - 1].s = s;
            ls = s;
            if (ps == s) err |= 4;  // the fold made the last vertex a non-kink: rare, bail out
            return;
        }
        if (out) out[m] = Vtx{x, f, s};
        m++;
        ps = have ? ls : NAN;
        have = true;
        lx = x;
        ls = s;
    }
};

// emission of z for the W vertex w and its right piece, shared by the count and
// write passes.  Returns z's slope at the end of the piece.
struct EmitAdapter {
    LEmit* e;
    __device__ __forceinline__ void push(double x, double f, double s) { e->push(x, f, s); }
};

static __device__ __noinline__ int node_update(const Fn U, const Fn D, double lo, double hi, double ux, double uf,
                                        bool seller, Vtx* scratch, int scap, Vtx* arena, int* counter, int acap,
                                        int& zoff, int& nZ, int lane) {
    const HCtx h = make_ctx(U, D);
    {
        const double sWr = h.wInf_U ? U.v(U.n - 1).s : D.v(D.n - 1).s;
        const double sWl = h.tailL_U ? U.sl : D.sl;
        if (sWr < lo || sWl > hi) return DEV_UNBOUNDED;
    }
    // segments: lane i owns events [k0, k1)
    const int nE = h.nE;
    const int k0 = (int)(((long long)nE * lane) / 32), k1 = (int)(((long long)nE * (lane + 1)) / 32);
    // ---- pass 1: W vertices of the segment: g / h minima, first vertex, local minima of g ----
    double gmin = INFINITY, hmin = INFINITY, fx = INFINITY, fg = INFINITY;
    int nw = 0;
    double lmx[LMAX], lmg[LMAX];  // local minima of g (x, g), in order
    int nlm = 0;
    int fail = 0;
    {
        WGen G;
        G.init(h, k0, k1, lane);
        WV w;
        double gprev = INFINITY, xprev = 0.0;
        bool desc = false;  // g was decreasing into the previous vertex
        while (G.next(w)) {
            const double g = fma(-lo, w.x, w.f), hh = fma(-hi, w.x, w.f);
            if (nw == 0) { fx = w.x; fg = g; }
            gmin = fmin(gmin, g);
            hmin = fmin(hmin, hh);
            // the previous vertex is a local minimum of g when g stops decreasing there
            if (nw > 0 && desc && !(g < gprev)) {
                if (nlm < LMAX) {
#pragma unroll
                    for (int i = 0; i < LMAX; ++i)
                        if (i == nlm) { lmx[i] = xprev; lmg[i] = gprev; }
                    nlm++;
                } else {
                    fail = 1;
                }
            }
            desc = nw > 0 ? (g < gprev) : true;
            gprev = g;
            xprev = w.x;
            nw++;
        }
        // the last vertex ends a descent: a local minimum within the lane
        if (nw > 0 && desc) {
            if (nlm < LMAX) {
#pragma unroll
                for (int i = 0; i < LMAX; ++i)
                    if (i == nlm) { lmx[i] = xprev; lmg[i] = gprev; }
                nlm++;
            } else {
                fail = 1;
            }
        }
    }
    // suffix minima over the recorded local minima (lmg[i] = min over i..nlm-1)
#pragma unroll
    for (int i = LMAX - 2; i >= 0; --i)
        if (i + 1 < nlm) lmg[i] = fmin(lmg[i], lmg[i + 1]);
    if (__any_sync(FULLM, fail))
        return node_update_chunk(U, D, lo, hi, ux, uf, seller, scratch, scap, arena, counter, acap, zoff, nZ, lane);
    // ---- scans ----
    const double Mr = excl_suffix_min(gmin, lane);   // g over later lanes
    const double Pl = excl_prefix_min(hmin, lane);   // h over earlier lanes
    // next W vertex after this lane: first vertex of the nearest later non-empty lane
    int nxt = nw > 0 ? lane : 32;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_down_sync(FULLM, nxt, o);
        if (lane + o < 32) nxt = min(nxt, y);
    }
    int nl = __shfl_down_sync(FULLM, nxt, 1);
    if (lane == 31) nl = 32;
    const double Xs = __shfl_sync(FULLM, fx, nl < 32 ? nl : 0);  // (every lane shuffles)
    const double Xr = nl < 32 ? Xs : INFINITY;
    int before;
    {
        int tot;
        before = excl_prefix_sum(nw > 0 ? 1 : 0, lane, tot);
    }
    const bool first_overall = before == 0 && nw > 0;
    const PCtx c{lo, hi, ux, uf, seller};

    // ---- pass 2 (twice: count, then write) ----
    int cnt = 0, drop = 0, off = 0, total = 0;
    double s_end = NAN, first_s = NAN;
    bool pend_first = false;
    bool folded_first = false;
    const int base = *counter;
    for (int pass = 0; pass < 2; ++pass) {
        LEmit E;
        // this lane's region starts at arena[base + off]; a dropped first candidate
        // would sit just before it and is never written
        E.out = pass ? arena + base + off - drop : nullptr;
        E.m = 0;
        E.have = false;
        E.ps = NAN;
        E.err = DEV_OK;
        WGen G;
        G.init(h, k0, k1, lane);
        WV w, wn;
        bool has = G.next(w);
        double P = Pl;
        double s_run = NAN;
        int li = 0;  // next local minimum index (by position)
        bool first = true;
        while (has) {
            const bool hasn = G.next(wn);
            const double xn = hasn ? wn.x : Xr;
            // M after w: g at the next W vertex, later local minima, later lanes
            while (li < nlm && !(lmx[li > LMAX - 1 ? LMAX - 1 : li] > w.x)) ++li;
            double Mnext = Mr;
            if (hasn) Mnext = fmin(Mnext, fma(-lo, wn.x, wn.f));
            if (li < nlm) {
                double lv = INFINITY;
#pragma unroll
                for (int i = 0; i < LMAX; ++i)
                    if (i == li) lv = lmg[i];
                Mnext = fmin(Mnext, lv);
            }
            const double Mj = fmin(fma(-lo, w.x, w.f), Mnext);
            LEmit* Ep = &E;
            EmitAdapter ad{Ep};
            if (first && first_overall) {
                const Line LW{w.x, w.f, w.sL}, LM{0.0, Mj, lo}, LP{0.0, INFINITY, hi};
                const double mv = LM.at(ux);
                const double tl = ftol(mv, uf);
                const bool zU0 = fabs(uf - mv) > tl ? (seller ? uf > mv : uf < mv) : false;
                s_run = emit_open(-INFINITY, w.x, LW, LM, true, LP, false, c, lo, zU0, ad);
            }
            int vi;
            bool zU;
            double zv;
            const double Pj = fmin(P, fma(-hi, w.x, w.f));
            const Line LWr{w.x, w.f, w.sR}, LMr{0.0, Mnext, lo}, LPr{0.0, Pj, hi};
            const double sr_ = z_side(LWr, LMr, isfinite(Mnext), LPr, true, c, w.x, true, vi, zU, zv);
            if (s_run != s_run) {  // unknown: checked against the left lane's slope
                if (pass == 0) { pend_first = E.m == 0; first_s = sr_; }
                if (!(pass == 1 && drop && E.m == 0 && !E.have)) E.push(w.x, zv, sr_);
                else { E.have = true; E.lx = w.x; E.ls = sr_; E.ps = NAN; E.m = 1; }
            } else if (sr_ != s_run) {
                E.push(w.x, zv, sr_);
            }
            s_run = emit_open(w.x, xn, LWr, LMr, isfinite(Mnext), LPr, true, c, sr_, false, ad);
            P = Pj;
            w = wn;
            has = hasn;
            first = false;
        }
        // a fold into a first vertex matters only when that vertex is dropped
        // (checked below, once drop is known)
        const bool fold8 = (E.err & 8) != 0;
        E.err &= ~8;
        if (__any_sync(FULLM, E.err))
            return node_update_chunk(U, D, lo, hi, ux, uf, seller, scratch, scap, arena, counter, acap, zoff, nZ,
                                     lane);
        if (pass == 0) {
            folded_first = fold8;
            cnt = E.m;
            s_end = s_run;
            // the slope arriving from the left: s_end of the nearest earlier non-empty lane
            int src = nw > 0 ? lane : -1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULLM, src, o);
                if (lane >= o) src = max(src, y);
            }
            int srcp = __shfl_up_sync(FULLM, src, 1);
            if (lane == 0) srcp = -1;
            const double se = __shfl_sync(FULLM, s_end, srcp < 0 ? 0 : srcp);
            const double s_left = srcp >= 0 ? se : lo;  // z's left tail slope is lo
            drop = (pend_first && !first_overall && first_s == s_left) ? 1 : 0;
            if (__any_sync(FULLM, drop && folded_first))
                return node_update_chunk(U, D, lo, hi, ux, uf, seller, scratch, scap, arena, counter, acap, zoff,
                                         nZ, lane);
            cnt -= drop;
            off = excl_prefix_sum(cnt, lane, total);
            if (base + total > acap) return DEV_OVERFLOW;
        }
    }
    __syncwarp();
    if (total == 0) {
        if (base + 1 > acap) return DEV_OVERFLOW;
        if (lane == 0) arena[base] = Vtx{0.0, fma(lo, -ux, uf), lo};
        total = 1;
    }
    if (lane == 0) *counter = base + total;
    __syncwarp();
    zoff = base;
    nZ = total;
    return DEV_OK;
}

// ===========================================================================
// Block-synchronous heavy update (the default tier 3).  No binary search and
// no dependent load chain touches global memory: every global access is a
// coalesced 32-wide load or store.
//   sweep A (left to right): the merged events of U and D in blocks of 32.
//     Lane i loads U[a+i] and D[b+i] into a per-warp shared window (cursors a,
//     b carried across blocks); each window element's merged position is its
//     index plus its rank in the other window (a 5-step binary search in
//     shared memory); lane k takes merged event k.  The vertices of W =
//     max(U, D) are compacted into the scratch buffer Wb.
//   sweep B (right to left over W in blocks of 32): Mafter[b] = min of
//     g = W - lo x over the blocks after b.
//   sweep C (left to right): lane i owns W vertex 32 b + i and emits z on its
//     right piece: v = min(W, lo y + M_{j+1}, hi y + P_j) (header identity),
//     z = OP(u, v); staging, de-duplication, folding and compaction as in
//     node_update_chunk.
// ===========================================================================
struct HWin {
    Vtx u[33], d[33];  // [0]: the vertex before the window (or the left-tail anchor); [1..32]: window
    int ev[32];        // merged event k of the block: isU | idx << 1 | rank << 7
};
static_assert(sizeof(HWin) >= 2 * 32 * sizeof(Vtx), "sweep C stages two rows in the windows");

__device__ __forceinline__ Vtx shfl_vtx(const Vtx& v, int src) {
    return Vtx{__shfl_sync(FULLM, v.x, src), __shfl_sync(FULLM, v.f, src), __shfl_sync(FULLM, v.s, src)};
}

template <bool RL = RL_DEFAULT>
__device__ __forceinline__ int rank_lt(const Vtx* w, double x) {  // #{m < 32 : w[1+m].x < x}
    int p = 0;
#pragma unroll(RL ? 1 : 5)
    for (int s = 16; s > 0; s >>= 1)
        if (w[p + s].x < x) p += s;  // w[p+s] = window element p+s-1
    return p + (w[p + 1].x < x ? 1 : 0);
}
template <bool RL = RL_DEFAULT>
__device__ __forceinline__ int rank_le(const Vtx* w, double x) {  // #{m < 32 : w[1+m].x <= x}
    int p = 0;
#pragma unroll(RL ? 1 : 5)
    for (int s = 16; s > 0; s >>= 1)
        if (w[p + s].x <= x) p += s;
    return p + (w[p + 1].x <= x ? 1 : 0);
}

// event k of the current block (window state in Wn); a, b: cursors (global
// indices of window element 0), for the left-slope of the first vertices
__device__ __forceinline__ Ev block_event(const HWin& Wn, int code) {
    Ev e;
    e.skip = false;
    const bool isU = code & 1;
    const int idx = (code >> 1) & 63, r = code >> 7;
    if (isU) {
        const Vtx V = Wn.u[1 + idx];
        e.x = V.x; e.eU = V.f; e.sUR = V.s; e.sUL = Wn.u[idx].s;
        const Vtx P = Wn.d[r];
        if (r < 32 && Wn.d[1 + r].x == e.x) {  // coincident vertices: one event
            const Vtx Q = Wn.d[1 + r];
            e.eD = Q.f; e.sDL = P.s; e.sDR = Q.s;
        } else {
            e.eD = fma(P.s, e.x - P.x, P.f); e.sDL = P.s; e.sDR = P.s;
        }
    } else {
        const Vtx V = Wn.d[1 + idx];
        e.x = V.x; e.eD = V.f; e.sDR = V.s; e.sDL = Wn.d[idx].s;
        const Vtx P = Wn.u[r];
        e.eU = fma(P.s, e.x - P.x, P.f); e.sUL = P.s; e.sUR = P.s;
        if (P.x == e.x) {  // the U vertex at the same x handled both (r = 0: the previous block's)
            e.skip = true;
            e.eU = P.f; e.sUR = P.s; e.sUL = P.s;  // sUL unused for a skip
        }
    }
    return e;
}

// z is written to zout[0 .. nZ) (contiguous, capacity zcap)
template <class WinPtr, bool RL = RL_DEFAULT>
static __device__ __noinline__ int node_update_block(const Fn U, const Fn D, double lo, double hi, double ux, double uf,
                                              bool seller, WinPtr win, Vtx* scratch, int scap, Vtx* zout, int zcap,
                                              int& nZ, int lane) {
    Vtx* const arena = zout;
    const int acap = zcap;
    HWin& Wn = *win;
    const HCtx h = make_ctx(U, D);
    {
        const double sWr = h.wInf_U ? U.v(U.n - 1).s : D.v(D.n - 1).s;
        const double sWl = h.tailL_U ? U.sl : D.sl;
        if (sWr < lo || sWl > hi) return DEV_UNBOUNDED;
    }
    const int nE = h.nE;
    const int wcap = 2 * nE + 8;  // W: at most a crossing and a vertex per event, plus the right tail
    const int nbmax = (wcap + 31) / 32;
    if ((size_t)scap < (size_t)STAGE * 32 + (size_t)wcap + (size_t)nbmax + 2) return DEV_OVERFLOW;
    (void)nbmax;
    Vtx* const stage_buf = scratch;
    Vtx* const Wb = scratch + STAGE * 32;
    double* const Mafter = reinterpret_cast<double*>(Wb + wcap);

    // ---- sweep A: W = max(U, D) into Wb ----
    int a = 0, b = 0, nW = 0;
    double cx = -INFINITY;   // x of the last event of the previous block
    bool cwr = h.tailL_U;    // winner just right of it (first block: the left-tail winner)
    const Vtx SENT{INFINITY, 0.0, 0.0};
    if (lane == 0) {
        Wn.u[0] = Vtx{U.v(0).x, U.v(0).f, U.sl};
        Wn.d[0] = Vtx{D.v(0).x, D.v(0).f, D.sl};
    }
    Wn.u[1 + lane] = (lane < U.n) ? U.v(lane) : SENT;
    Wn.d[1 + lane] = (lane < D.n) ? D.v(lane) : SENT;
    // software pipeline: the 32 elements after each window are loaded one block
    // ahead (registers), so no block waits on global memory
    Vtx pu = (32 + lane < U.n) ? U.v(32 + lane) : SENT;
    Vtx pd = (32 + lane < D.n) ? D.v(32 + lane) : SENT;
    __syncwarp();
    for (int k0 = 0; k0 < nE; k0 += 32) {
        const int nrem = min(32, nE - k0);
        {
            const Vtx uu = Wn.u[1 + lane], dd = Wn.d[1 + lane];
            if (a + lane < U.n) {
                const int r = rank_lt<RL>(Wn.d, uu.x);
                const int pos = lane + r;
                if (pos < nrem) Wn.ev[pos] = 1 | (lane << 1) | (r << 7);
            }
            if (b + lane < D.n) {
                const int r = rank_le<RL>(Wn.u, dd.x);
                const int pos = lane + r;
                if (pos < nrem) Wn.ev[pos] = (lane << 1) | (r << 7);
            }
        }
        __syncwarp();
        const bool valid = lane < nrem;
        const int code = valid ? Wn.ev[lane] : 0;
        Ev e;
        if (valid) e = block_event(Wn, code);
        else { e.x = INFINITY; e.eU = e.eD = 0.0; e.sUL = e.sUR = e.sDL = e.sDR = 0.0; e.skip = true; }
        const bool wr = valid ? winR(e) : false;
        double x_prev = __shfl_up_sync(FULLM, e.x, 1);
        bool wRp = __shfl_up_sync(FULLM, (int)wr, 1) != 0;
        if (lane == 0) { x_prev = cx; wRp = cwr; }
        // W's vertices of this event (as w_vertices), written straight to Wb: only
        // the flags and the two crossing positions live across the prefix sum, and
        // one vertex at a time is built for its store (the WV3 of w_vertices cost
        // ~40 registers here and spilled around every block)
        bool h0 = false, h1 = false, h2 = false;
        double y0 = 0.0, y2 = 0.0;
        bool wl = false;
        if (valid && !e.skip) {
            wl = winL(e);
            if (wRp != wl) {  // crossing on (x_prev, x)
                const double e_w = wl ? e.eU : e.eD, e_o = wl ? e.eD : e.eU;
                const double s_w = wl ? e.sUL : e.sDL, s_o = wl ? e.sDL : e.sUL;
                if (s_w != s_o) {
                    y0 = e.x - (e_w - e_o) / (s_w - s_o);
                    h0 = y0 > x_prev && y0 < e.x;
                }
            }
            h1 = (wl ? e.sUL : e.sDL) != (wr ? e.sUR : e.sDR);
            if (k0 + lane == h.klast && wr != h.wInf_U) {  // crossing on (x, +inf)
                const double e_w = wr ? e.eU : e.eD, e_o = wr ? e.eD : e.eU;
                const double s_w = wr ? e.sUR : e.sDR, s_o = wr ? e.sDR : e.sUR;
                if (s_o != s_w) {
                    y2 = e.x + (e_w - e_o) / (s_o - s_w);
                    h2 = y2 > e.x;
                }
            }
        }
        int tot;
        const int off = excl_prefix_sum_bits<2>((int)h0 + (int)h1 + (int)h2, lane, tot);  // <= 3
        if (nW + tot > wcap) return DEV_FALLBACK;  // cannot happen
        {
            Vtx* o = Wb + nW + off;
            if (h0) {
                const double e_w = wl ? e.eU : e.eD, s_w = wl ? e.sUL : e.sDL;
                *o++ = Vtx{y0, fma(s_w, y0 - e.x, e_w), s_w};
            }
            if (h1) *o++ = Vtx{e.x, fmax(e.eU, e.eD), wr ? e.sUR : e.sDR};
            if (h2) {
                const double e_w = wr ? e.eU : e.eD, s_w = wr ? e.sUR : e.sDR, s_o = wr ? e.sDR : e.sUR;
                *o = Vtx{y2, fma(s_w, y2 - e.x, e_w), s_o};
            }
        }
        nW += tot;
        const unsigned bu = __ballot_sync(FULLM, valid && (code & 1));
        const unsigned bv = __ballot_sync(FULLM, valid);
        const int cU = __popc(bu), cD = __popc(bv) - cU;
        cx = __shfl_sync(FULLM, e.x, 31);
        cwr = __shfl_sync(FULLM, (int)wr, 31) != 0;
        // shift the windows by the consumed elements, refill from the prefetch
        {
            const Vtx pu_s = shfl_vtx(pu, (lane + cU) & 31), pd_s = shfl_vtx(pd, (lane + cD) & 31);
            const Vtx nu = (lane + cU < 32) ? Wn.u[1 + lane + cU] : pu_s;
            const Vtx nd = (lane + cD < 32) ? Wn.d[1 + lane + cD] : pd_s;
            const Vtx pvu = Wn.u[cU], pvd = Wn.d[cD];
            __syncwarp();
            Wn.u[1 + lane] = nu;
            Wn.d[1 + lane] = nd;
            if (lane == 0) {
                Wn.u[0] = pvu;
                Wn.d[0] = pvd;
            }
        }
        a += cU;
        b += cD;
        pu = (a + 32 + lane < U.n) ? U.v(a + 32 + lane) : SENT;
        pd = (b + 32 + lane < D.n) ? D.v(b + 32 + lane) : SENT;
        __syncwarp();
    }
    if (nW == 0) return DEV_FALLBACK;  // W is a line: not a heavy node (caller falls back)
    const double slW = h.tailL_U ? U.sl : D.sl;
    const int nb = (nW + 31) / 32;

    // ---- sweep B: Mafter[b] = min of g over blocks > b ----
    {
        double Mc = INFINITY;
        int j = (nb - 1) * 32 + lane;
        Vtx v = (j < nW) ? Wb[j] : SENT;
        for (int blk = nb - 1; blk >= 0; --blk) {
            const Vtx vn = (blk > 0) ? Wb[j - 32] : SENT;  // prefetch the block to the left
            const double g = (j < nW) ? fma(-lo, v.x, v.f) : INFINITY;
            if (lane == 0) Mafter[blk] = Mc;
            Mc = fmin(Mc, warp_min<RL>(g));
            v = vn;
            j -= 32;
        }
    }
    __syncwarp();

    // ---- sweep C: z on every piece of W ----
    const PCtx c{lo, hi, ux, uf, seller};
    const int base = 0;
    int total = 0;
    int err = DEV_OK;
    double Pc = INFINITY;
    double s_in = lo;           // z's slope arriving from the left (z's left tail is lo)
    double last_x = -INFINITY;  // the last vertex written (earlier blocks)
    Vtx wv_nx = (lane < nW) ? Wb[lane] : SENT;
    double prev_s = slW;  // slope right of the last W vertex of the previous block
    for (int blk = 0; blk < nb; ++blk) {
        const int j = blk * 32 + lane;
        const bool has = j < nW;
        const Vtx wv = wv_nx;
        wv_nx = (j + 32 < nW) ? Wb[j + 32] : SENT;  // prefetch the next block
        double sL = __shfl_up_sync(FULLM, wv.s, 1);
        if (lane == 0) sL = prev_s;
        prev_s = __shfl_sync(FULLM, wv.s, 31);
        double xn = __shfl_down_sync(FULLM, wv.x, 1);
        const double xn31 = __shfl_sync(FULLM, wv_nx.x, 0);
        if (lane == 31) xn = xn31;
        const double gl = has ? fma(-lo, wv.x, wv.f) : INFINITY;
        const double hl = has ? fma(-hi, wv.x, wv.f) : INFINITY;
        const double Mnext = fmin(excl_suffix_min<RL>(gl, lane), Mafter[blk]);  // g over later W vertices
        const double hpre = excl_prefix_min<RL>(hl, lane);
        const double Pl = fmin(hpre, Pc);                                   // h over earlier W vertices
        const bool first_overall = has && j == 0;
        Stage st;
        st.buf = stage_buf;
        st.sbuf = reinterpret_cast<Vtx*>(&Wn);  // the merge windows are dead in sweep C: 2 stage rows
        st.lane = lane;
        st.m = 0;
        st.err = DEV_OK;
        st.last_s = NAN;
        double s_run = NAN;
        bool pending = false;
        const double Pj = fmin(Pl, hl);
        const bool fast = has && !first_overall && piece_is_w(wv.x, wv.f, wv.s, xn, Mnext, Pj, c);
        AMTC_HEAVY_STAT(has ? (fast ? 1 : 2) : 0);
#ifdef AMTC_HEAVY_STAT_BLOCKS
        if (__ballot_sync(FULLM, has && !fast) == 0u && lane == 0) AMTC_HEAVY_STAT(3);
#endif
        if (fast) {
            pending = true;
            st.push(wv.x, wv.f, wv.s);
            s_run = wv.s;
        } else if (has) {
#ifdef AMTC_SWEEPC_MERGED
            // One inlined copy of emit_open serves both the left tail (ph = 0: only
            // W's first vertex, once per node) and the vertex's right piece (ph = 1):
            // two copies made the loop body ~35 KB of code, more than the 32 KB
            // instruction cache level shared by the SM's warps (half of all stall
            // samples are instruction-fetch stalls, profiles/r02_ncu_source_calls_N400.txt)
#pragma unroll 1
            for (int ph = first_overall ? 0 : 1; ph < 2; ++ph) {
                Line LWq, LMq, LPq;
                bool hasMq, hasPq, zUq;
                double aq, bq, sq;
                int viq;
                if (ph == 0) {
                    const double Mj = fmin(gl, Mnext);
                    LWq = Line{wv.x, wv.f, sL};
                    LMq = Line{0.0, Mj, lo};
                    LPq = Line{0.0, INFINITY, hi};
                    const double mv = LMq.at(ux);
                    const double tl = ftol(mv, uf);
                    zUq = fabs(uf - mv) > tl ? (seller ? uf > mv : uf < mv) : false;
                    hasMq = true; hasPq = false;
                    aq = -INFINITY; bq = wv.x; sq = lo; viq = -1;
                } else {
                    LWq = Line{wv.x, wv.f, wv.s};
                    LMq = Line{0.0, Mnext, lo};
                    LPq = Line{0.0, Pj, hi};
                    hasMq = isfinite(Mnext); hasPq = true;
                    double zv;
                    const double sr_ = z_side(LWq, LMq, hasMq, LPq, true, c, wv.x, true, viq, zUq, zv);
                    const bool unknown = s_run != s_run;
                    if (unknown) pending = st.m == 0;
                    if (unknown || sr_ != s_run) st.push(wv.x, zv, sr_);
                    aq = wv.x; bq = xn; sq = sr_;
                }
                s_run = emit_open<Stage, true>(aq, bq, LWq, LMq, hasMq, LPq, hasPq, c, sq, zUq, st, viq);
            }
#else
            const double Mj = fmin(gl, Mnext);
            if (first_overall) {
                const Line LW{wv.x, wv.f, sL}, LM{0.0, Mj, lo}, LP{0.0, INFINITY, hi};
                const double mv = LM.at(ux);
                const double tl = ftol(mv, uf);
                const bool zU0 = fabs(uf - mv) > tl ? (seller ? uf > mv : uf < mv) : false;
                s_run = emit_open<Stage, AMTC_ENTRY_KNOWN_V>(-INFINITY, wv.x, LW, LM, true, LP, false, c, lo, zU0, st);
            }
            int vi;
            bool zU;
            double zv;
            const Line LWr{wv.x, wv.f, wv.s}, LMr{0.0, Mnext, lo}, LPr{0.0, Pj, hi};
            const double sr_ = z_side(LWr, LMr, isfinite(Mnext), LPr, true, c, wv.x, true, vi, zU, zv);
            if (s_run != s_run) {
                pending = st.m == 0;
                st.push(wv.x, zv, sr_);
            } else if (sr_ != s_run) {
                st.push(wv.x, zv, sr_);
            }
            s_run = emit_open<Stage, AMTC_ENTRY_KNOWN_V>(wv.x, xn, LWr, LMr, isfinite(Mnext), LPr, true, c, sr_, zU, st, vi);
#endif
        }
        const double s_end = s_run;
        // the slope arriving from the left: s_end of the previous lane (all lanes
        // below the last valid one hold a vertex), or of the previous block
        double s_left = __shfl_up_sync(FULLM, s_end, 1);
        if (lane == 0) s_left = s_in;
        {
            const int lastv = min(31, nW - 1 - blk * 32);
            s_in = __shfl_sync(FULLM, s_end, lastv);
        }
        const int skip0 = (pending && st.at(0).s == s_left) ? 1 : 0;
        if (__reduce_or_sync(FULLM, st.err)) { err = DEV_FALLBACK; break; }  // stage overflow
        int cnt = st.m - skip0;
        double f0x = 0.0, fs = 0.0, lx = -INFINITY;
        if (cnt > 0) {
            f0x = st.at(skip0).x;
            fs = st.at(skip0).s;
            lx = st.at(st.m - 1).x;
        }
        int prevl = cnt > 0 ? lane : -1;
        int nextl = cnt > 0 ? lane : 32;
#pragma unroll(RL ? 1 : 5)
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULLM, prevl, o);
            if (lane >= o) prevl = max(prevl, y);
            const int z = __shfl_down_sync(FULLM, nextl, o);
            if (lane + o < 32) nextl = min(nextl, z);
        }
        int pl = __shfl_up_sync(FULLM, prevl, 1);
        if (lane == 0) pl = -1;
        int nl = __shfl_down_sync(FULLM, nextl, 1);
        if (lane == 31) nl = 32;
        const double px = __shfl_sync(FULLM, lx, pl < 0 ? 0 : pl);
        const double prev_x = pl < 0 ? last_x : px;
        const bool fold = cnt > 0 && !(f0x > prev_x + xtol(f0x));
        const int nfold = __shfl_sync(FULLM, (int)fold, nl > 31 ? 0 : nl);
        const double nfs = __shfl_sync(FULLM, fs, nl > 31 ? 0 : nl);
        if (cnt > 0 && nl <= 31 && nfold) st.at(st.m - 1).s = nfs;
        if (fold && pl < 0 && total > 0) arena[base + total - 1].s = fs;
        const int drop_first = (fold && (pl >= 0 || total > 0)) ? 1 : 0;
        cnt -= drop_first;
        int tot;
        static_assert(STAGE < 64, "cnt < 2^6");
        const int off = excl_prefix_sum_bits<6>(cnt, lane, tot);  // 0 <= cnt <= STAGE
        if (base + total + tot > acap) { err = DEV_OVERFLOW; break; }
        for (int q = 0; q < cnt; ++q)
            arena[base + total + off + q] = st.at(q + skip0 + drop_first);
        total += tot;
        {
            const int lastl = __shfl_sync(FULLM, prevl, 31);
            const double lxl = __shfl_sync(FULLM, lx, lastl < 0 ? 0 : lastl);
            if (lastl >= 0) last_x = lxl;
        }
        Pc = fmin(Pc, __shfl_sync(FULLM, fmin(hpre, hl), 31));
        __syncwarp();
    }
    if (err) return err;
    if (total == 0) {
        if (base + 1 > acap) return DEV_OVERFLOW;
        if (lane == 0) arena[base] = Vtx{0.0, fma(lo, -ux, uf), lo};
        total = 1;
    }
    __syncwarp();
    nZ = total;
    return DEV_OK;
}

// a6 helper: the value at y = 0 of the restriction of W = max(U, D) to slopes
// [lo, hi] (t = 0; lo = hi = -S0 without costs at t = 0):
//   v_0(0) = min( W(0), min_{x_j >= 0} W_j - lo x_j, min_{x_j <= 0} W_j - hi x_j )
// (buying up to a position x_j >= 0 at the ask -lo, selling down at the bid -hi;
// infima of PWL functions over half lines sit at 0 or at vertices).  Also W's
// tail slopes (boundedness) and the minimising vertex (the root hedge, smallest
// x on ties).
static __device__ __noinline__ double root_min(const Fn U, const Fn D, double lo, double hi, double& slW, double& srW,
                                        double& ymin, int lane) {
    const HCtx h = make_ctx(U, D);
    const int nb = (h.nE + 31) / 32;
    double mv = INFINITY, mx = INFINITY;    // best vertex value and position
    double lx = -INFINITY, lval = INFINITY;  // the last vertex at or left of 0: W(0) from its right piece
    double fx = INFINITY, fval = 0.0;       // the first vertex (W(0) from the left tail if none <= 0)
    for (int blk = 0; blk < nb; ++blk) {
        const BlockW B = block_w(h, blk, lane);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (q >= B.w.n) break;
            const WV w = B.w.get(q);
            if (w.x >= 0.0) {
                const double g = fma(-lo, w.x, w.f);
                if (g < mv || (g == mv && w.x < mx)) { mv = g; mx = w.x; }
            }
            if (w.x <= 0.0) {
                const double g = fma(-hi, w.x, w.f);
                if (g < mv || (g == mv && w.x < mx)) { mv = g; mx = w.x; }
                if (w.x > lx) { lx = w.x; lval = fma(w.sR, -w.x, w.f); }
            }
            if (w.x < fx) { fx = w.x; fval = fma(w.sL, -w.x, w.f); }
        }
    }
    slW = h.tailL_U ? U.sl : D.sl;
    srW = h.wInf_U ? U.v(U.n - 1).s : D.v(D.n - 1).s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(FULLM, mv, o), ox = __shfl_xor_sync(FULLM, mx, o);
        if (ov < mv || (ov == mv && ox < mx)) { mv = ov; mx = ox; }
        const double olx = __shfl_xor_sync(FULLM, lx, o), olv = __shfl_xor_sync(FULLM, lval, o);
        if (olx > lx) { lx = olx; lval = olv; }
        const double ofx = __shfl_xor_sync(FULLM, fx, o), ofv = __shfl_xor_sync(FULLM, fval, o);
        if (ofx < fx) { fx = ofx; fval = ofv; }
    }
    const double w0 = (lx > -INFINITY) ? lval : fval;  // W(0)
    ymin = mx;
    if (w0 < mv) { mv = w0; ymin = 0.0; }
    return mv;
}

}  // namespace heavy
}  // namespace amtc
