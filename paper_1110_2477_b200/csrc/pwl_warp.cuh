// pwl_warp.cuh -- warp-cooperative node update for HEAVY node functions
// (thousands of vertices: the buyer's "sawtooth" ridge of calls / bull spreads
// at large k/h).
//
// Data-parallel reformulation of the node recursion.  With
// W = max(z^u, z^d) (discounted) and the restriction to [lo, hi]
// (reading R7):
//     A(y) = inf_{y'>=y} W(y') + lo (y - y') = min( W(y), lo y + M(y) ),
//     B(y) = inf_{y'<=y} W(y') + hi (y - y') = min( W(y), hi y + P(y) ),
//     M(y) = min over vertices x_k >= y of (W_k - lo x_k)   (suffix minimum),
//     P(y) = min over vertices x_k <= y of (W_k - hi x_k)   (prefix minimum),
// because an infimum of a PWL function over a half line is attained at the end
// point or at a vertex (the tails are monotone when d < r < u).  So
//     v = min(A, B) = min( W, lo y + M, hi y + P )
// and on every piece of W both M and P are constants: v is the lower envelope
// of at most three lines there, and z = max(u, v) (seller) / min(u, v)
// (buyer) adds at most the two lines of u.  Hence:
//   1. W by a merge-path split of the two children over the 32 lanes;
//   2. suffix-min / prefix-min scans (lane-chunked + warp shuffles);
//   3. every piece of W emits its vertices of z independently;
//   4. warp prefix sums compact the per-lane outputs.
#pragma once
#include "pwl_device.cuh"

namespace amtc {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(FULL, x, 31);
    return x - v;
}

// (value, x, f) record whose minimum is taken on value
struct MinRec {
    double v, x, f;
};

__device__ __forceinline__ MinRec minrec(const MinRec& a, const MinRec& b) { return (b.v < a.v) ? b : a; }

__device__ __forceinline__ MinRec shfl_rec_up(const MinRec& r, int o) {
    return MinRec{__shfl_up_sync(FULL, r.v, o), __shfl_up_sync(FULL, r.x, o), __shfl_up_sync(FULL, r.f, o)};
}
__device__ __forceinline__ MinRec shfl_rec_down(const MinRec& r, int o) {
    return MinRec{__shfl_down_sync(FULL, r.v, o), __shfl_down_sync(FULL, r.x, o), __shfl_down_sync(FULL, r.f, o)};
}

// number of U vertices among the first k of the merged order (U first on ties)
__device__ __forceinline__ int merge_split(const Fn& U, const Fn& D, int k) {
    int lo = max(0, k - D.n), hi = min(k, U.n);
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (U.v(mid).x <= D.v(k - mid - 1).x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// copy `m` vertices from a lane region into a compact array at offset `o`
__device__ __forceinline__ void copy_vtx(Vtx* dst, const Vtx* src, int m) {
    for (int i = 0; i < m; ++i) dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// stage 1: W = max(U, D), lanes own contiguous ranges of merged events
// ---------------------------------------------------------------------------
__device__ __forceinline__ int warp_merge_max(const Fn& F, const Fn& G, Vtx* raw, Vtx* W, int wcap, int& nW,
                                              double& slW, int lane) {
    const int nE = F.n + G.n;
    const int per = (nE + 31) / 32;
    const int k0 = min(lane * per, nE), k1 = min(k0 + per, nE);
    // reconstruct the sequential sweep state just before event k0
    int iF = merge_split(F, G, k0) - 1;
    int iG = (k0 - (iF + 1)) - 1;
    double sF = F.slope_right(iF), sG = G.slope_right(iG);
    bool curF;
    double xprev, eF, eG;
    {
        double xe0 = fmin(F.v(0).x, G.v(0).x);
        double eF0 = piece_at(F, -1, xe0), eG0 = piece_at(G, -1, xe0);
        if (F.sl != G.sl) curF = F.sl < G.sl;
        else curF = eF0 >= eG0;
        slW = curF ? F.sl : G.sl;
    }
    if (k0 > 0) {
        xprev = fmax(iF >= 0 ? F.v(iF).x : -INFINITY, iG >= 0 ? G.v(iG).x : -INFINITY);
        eF = (iF >= 0 && F.v(iF).x == xprev) ? F.v(iF).f : piece_at(F, iF, xprev);
        eG = (iG >= 0 && G.v(iG).x == xprev) ? G.v(iG).f : piece_at(G, iG, xprev);
        if (fabs(eF - eG) > ftol(eF, eG)) curF = eF > eG;
        else curF = sF >= sG;
    } else {
        xprev = -INFINITY;
        eF = eG = 0.0;
    }
    Vtx* mine = raw + 2 * k0 + 2 * lane;
    Emit E;
    E.init(mine, 2 * (k1 - k0) + 2, curF ? sF : sG);
    double xe = xprev;
    for (int k = k0; k < k1; ++k) {
        double xF = (iF + 1 < F.n) ? F.v(iF + 1).x : INFINITY;
        double xG = (iG + 1 < G.n) ? G.v(iG + 1).x : INFINITY;
        // merged order takes F first on ties: exactly one vertex per event
        const bool takeF = xF <= xG;
        xe = takeF ? xF : xG;
        eF = (takeF) ? F.v(iF + 1).f : piece_at(F, iF, xe);
        eG = (!takeF) ? G.v(iG + 1).f : piece_at(G, iG, xe);
        const double tl = ftol(eF, eG);
        bool lost = curF ? (eG > eF + tl) : (eF > eG + tl);
        if (lost) {
            double yc = (sF != sG) ? xe - (eF - eG) / (sF - sG) : xe;
            yc = fmin(fmax(yc, xprev), xe);
            curF = !curF;
            double fc = curF ? piece_at(F, iF, yc) : piece_at(G, iG, yc);
            E.push(yc, fc, curF ? sF : sG);
        }
        if (takeF) { iF++; sF = F.v(iF).s; }
        else { iG++; sG = G.v(iG).s; }
        if (fabs(eF - eG) > tl) curF = eF > eG;
        else curF = sF >= sG;
        E.push(xe, fmax(eF, eG), curF ? sF : sG);
        xprev = xe;
    }
    if (k1 == nE && k0 < k1) {  // right tails
        double sw = curF ? sF : sG, sLo = curF ? sG : sF;
        double fw = curF ? eF : eG, fLo = curF ? eG : eF;
        if (sLo > sw) {
            double yc = xe + (fw - fLo) / (sLo - sw);
            if (!(yc >= xe)) yc = xe;
            E.push(yc, fma(sLo, yc - xe, fLo), sLo);
        }
    }
    int err = __reduce_or_sync(FULL, E.err);
    if (err) return err;
    int total;
    int off = warp_excl_scan(E.m, lane, total);
    if (total + 1 > wcap) return DEV_OVERFLOW;
    __syncwarp();
    copy_vtx(W + off, mine, E.m);
    if (total == 0 && lane == 0) {  // both children are one line: anchor
        W[0].x = F.v(0).x;
        W[0].f = fmax(F.v(0).f, piece_at(G, -1, F.v(0).x));
        W[0].s = slW;
    }
    nW = total == 0 ? 1 : total;
    __syncwarp();
    return DEV_OK;
}

// ---------------------------------------------------------------------------
// stage 3 helper: emit the vertices of z = OP(u, min(lines)) on (a, b)
// ---------------------------------------------------------------------------
struct Line {
    double x0, f0, s;
    __device__ __forceinline__ double at(double y) const { return fma(s, y - x0, f0); }
};

// z = OP(u, V) on the sub-interval (p, q) where V and u are single lines
__device__ __forceinline__ void emit_uv(double p, double q, const Line& V, const Line& Uq, bool seller, Emit& E) {
    // winner at p (p may be -inf: decide by slope)
    bool vwins;
    double vp = 0.0, up = 0.0;
    if (p == -INFINITY) {
        if (V.s != Uq.s) vwins = seller ? (V.s < Uq.s) : (V.s > Uq.s);
        else {
            double r = isfinite(q) ? q : V.x0;
            vwins = seller ? (V.at(r) >= Uq.at(r)) : (V.at(r) <= Uq.at(r));
        }
    } else {
        vp = V.at(p);
        up = Uq.at(p);
        if (fabs(vp - up) > ftol(vp, up)) vwins = seller ? (vp > up) : (vp < up);
        else vwins = seller ? (V.s >= Uq.s) : (V.s <= Uq.s);
        E.push(p, seller ? fmax(vp, up) : fmin(vp, up), vwins ? V.s : Uq.s);
    }
    // crossing inside (p, q): the loser overtakes
    const Line& Wn = vwins ? V : Uq;
    const Line& Lo = vwins ? Uq : V;
    if (Wn.s == Lo.s) return;
    bool better = seller ? (Lo.s > Wn.s) : (Lo.s < Wn.s);
    if (!better) return;
    // crossing y: Wn(y) = Lo(y)
    double yc;
    {
        double r = (p == -INFINITY) ? Wn.x0 : p;
        double d = Wn.at(r) - Lo.at(r);
        yc = r + d / (Lo.s - Wn.s);
    }
    if (!(yc < q)) return;
    if (p != -INFINITY && !(yc > p)) yc = p;
    E.push(yc, Lo.at(yc), Lo.s);
}

// v on (a, b) = lower envelope of lines[0..nl); then OP with u (vertex ux,uf; slopes lo|hi)
__device__ __forceinline__ void emit_piece(double a, double b, const Line* lines, int nl, double ux, double uf,
                                           double lo, double hi, bool seller, Emit& E) {
    // active line just right of a
    int act = 0;
    if (a == -INFINITY) {
        for (int l = 1; l < nl; ++l) {
            if (lines[l].s > lines[act].s) act = l;
            else if (lines[l].s == lines[act].s) {
                double r = isfinite(b) ? b : lines[l].x0;
                if (lines[l].at(r) < lines[act].at(r)) act = l;
            }
        }
    } else {
        double va = lines[0].at(a);
        for (int l = 1; l < nl; ++l) {
            double vl = lines[l].at(a);
            if (vl < va - ftol(vl, va) || (fabs(vl - va) <= ftol(vl, va) && lines[l].s < lines[act].s)) {
                act = l;
                va = vl;
            }
        }
    }
    double cur = a;
    for (int seg = 0; seg < 4; ++seg) {
        // next switch: a line with a smaller slope crossing below the active one
        double nxt = b;
        int nl_ = -1;
        for (int l = 0; l < nl; ++l) {
            if (l == act || !(lines[l].s < lines[act].s)) continue;
            double r = (cur == -INFINITY) ? lines[act].x0 : cur;
            double d = lines[l].at(r) - lines[act].at(r);
            double y = r + d / (lines[act].s - lines[l].s);  // where line l meets act
            if (cur != -INFINITY && !(y > cur)) y = cur;      // already (tie-)below: switch now
            if (y < nxt || (y == nxt && nl_ >= 0 && lines[l].s < lines[nl_].s)) {
                nxt = y;
                nl_ = l;
            }
        }
        const double q = (nl_ >= 0) ? nxt : b;
        // combine the v-segment (cur, q) with u, split at ux
        const Line& V = lines[act];
        Line UL{ux, uf, lo}, UR{ux, uf, hi};
        if (ux > cur && ux < q) {
            emit_uv(cur, ux, V, UL, seller, E);
            emit_uv(ux, q, V, UR, seller, E);
        } else {
            emit_uv(cur, q, V, (q <= ux) ? UL : UR, seller, E);
        }
        if (nl_ < 0) break;
        cur = q;
        act = nl_;
    }
}

// ---------------------------------------------------------------------------
// the warp-cooperative node update
// scratch: >= 22 * (U.n + D.n) + 2300 vertices; Z is appended to `arena`
// (bump counter `counter`, shared memory) at offset zoff
// ---------------------------------------------------------------------------
__device__ __noinline__ int warp_node_update(const Fn& U, const Fn& D, double lo, double hi, double ux, double uf,
                                             bool seller, Vtx* scratch, int scap, Vtx* arena, int* counter,
                                             int arena_cap, int& zoff, int& nZ, int lane) {
    const int nE = U.n + D.n;
    Vtx* raw = scratch;                  // 2 nE + 64
    Vtx* W = raw + (2 * nE + 64);        // 2 nE + 2
    Vtx* Ms = W + (2 * nE + 2);          // nW records (v, x, f) of the suffix minimum
    Vtx* zraw = Ms + (2 * nE + 2);       // 6 per piece + 64 per lane
    const int used_before_z = (int)(zraw - scratch);
    if (used_before_z >= scap) return DEV_OVERFLOW;
    int nW;
    double slW;
    int err = warp_merge_max(U, D, raw, W, 2 * nE + 2, nW, slW, lane);
    if (err) return err;
    // restriction is finite iff W's tails are steeper than the quotes (d < r < u)
    if (W[nW - 1].s < lo || slW > hi) return DEV_UNBOUNDED;

    // stage 2: chunked suffix-min of g = W - lo x and prefix-min of h = W - hi x
    const int per = (nW + 31) / 32;
    const int c0 = min(lane * per, nW), c1 = min(c0 + per, nW);
    const MinRec INF{INFINITY, 0.0, 0.0};
    MinRec gmin = INF, hmin = INF;
    for (int i = c0; i < c1; ++i) {
        MinRec g{fma(-lo, W[i].x, W[i].f), W[i].x, W[i].f};
        MinRec h{fma(-hi, W[i].x, W[i].f), W[i].x, W[i].f};
        gmin = minrec(gmin, g);
        if (h.v < hmin.v) hmin = h;
    }
    // exclusive suffix over lanes > lane (for g) and prefix over lanes < lane (for h)
    MinRec sufx = INF, pref = INF;
    {
        MinRec x = gmin;  // inclusive suffix scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            MinRec y = shfl_rec_down(x, o);
            if (lane + o < 32) x = minrec(x, y);
        }
        MinRec nxt = shfl_rec_down(x, 1);
        sufx = (lane < 31) ? nxt : INF;
        MinRec z = hmin;  // inclusive prefix scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            MinRec y = shfl_rec_up(z, o);
            if (lane >= o) z = minrec(y, z);
        }
        MinRec prv = shfl_rec_up(z, 1);
        pref = (lane > 0) ? prv : INF;
    }
    // per-vertex suffix minima of the chunk (Ms[i] = min over k >= i)
    {
        MinRec run = sufx;
        for (int i = c1 - 1; i >= c0; --i) {
            MinRec g{fma(-lo, W[i].x, W[i].f), W[i].x, W[i].f};
            run = minrec(g, run);
            Ms[i].x = run.v;
            Ms[i].f = run.x;
            Ms[i].s = run.f;
        }
    }
    __syncwarp();
    // stage 3: pieces i in [c0, c1) (lane 0 also the left tail, i = -1)
    const int pbeg = (lane == 0) ? -1 : c0;
    const int npieces = (c1 > c0 || lane == 0) ? (c1 - pbeg) : 0;
    const int zbase = 8 * (c0 + 1) + 64 * lane;  // lane region: 8 per piece + slack
    Vtx* mine = zraw + zbase;
    const int mycap = 8 * npieces + 8;
    if (used_before_z + zbase + mycap > scap) err = DEV_OVERFLOW;
    Emit E;
    // z's left tail is the quote slope lo (A.3: every z has tails lo / hi); the
    // other lanes start from "unknown" (NaN never equals a slope, so at worst
    // one redundant vertex per lane is kept; it vanishes at the next merge)
    E.init(mine, mycap, lane == 0 ? lo : NAN);
    MinRec P = pref;
    if (!err) {
        for (int i = pbeg; i < c1; ++i) {
            if (i >= 0) {
                MinRec h{fma(-hi, W[i].x, W[i].f), W[i].x, W[i].f};
                if (h.v < P.v) P = h;
            }
            // M for this piece: min over vertices >= i+1
            MinRec M;
            if (i + 1 < c1) M = MinRec{Ms[i + 1].x, Ms[i + 1].f, Ms[i + 1].s};
            else M = sufx;
            const double a = (i < 0) ? -INFINITY : W[i].x;
            const double b = (i + 1 < nW) ? W[i + 1].x : INFINITY;
            Line lines[3];
            int nl = 0;
            const Vtx& anc = W[i < 0 ? 0 : i];
            lines[nl++] = Line{anc.x, anc.f, i < 0 ? slW : anc.s};
            if (M.v < INFINITY) lines[nl++] = Line{M.x, M.f, lo};
            if (P.v < INFINITY) lines[nl++] = Line{P.x, P.f, hi};
            emit_piece(a, b, lines, nl, ux, uf, lo, hi, seller, E);
        }
    }
    err |= __reduce_or_sync(FULL, E.err | err);
    if (err) return err;
    int total;
    int off = warp_excl_scan(E.m, lane, total);
    if (total == 0) return DEV_OVERFLOW;  // (a line never reaches this path)
    int base = 0;
    if (lane == 0) base = atomicAdd(counter, total);
    base = __shfl_sync(FULL, base, 0);
    if (base + total > arena_cap) return DEV_OVERFLOW;
    copy_vtx(arena + base + off, mine, E.m);
    zoff = base;
    nZ = total;
    __syncwarp();
    return DEV_OK;
}

}  // namespace amtc
