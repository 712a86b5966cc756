// amtc_full.cu -- the FULL transaction-cost solver for the batched path: one
// warp per work item (option, party) whose node functions may grow large (the
// buyer of a call or a bull spread and the seller of a bull spread: the
// "sawtooth" of DESIGN.md section 5), swept in 32-column strips right to left
// (Sec. 3, on the tree of Sec. 4.1; region-B
// dependency P:164-166).
//
// It is the light solver's strip loop (amtc_light.cu: one shared-memory strip
// matrix whose columns 32 / 33 hold the carry column of the strip to the
// right, the carry record prefetched a level ahead, node quotes carried by one
// multiply per level) extended with the three storage tiers of a function:
//   * <= C vertices: a column of the strip matrix (the common case; both
//     children there -> the node update runs with compile-time strides);
//   * more: the warp's row arena in global memory (ping-pong by level parity),
//     updated by the lane itself (tier 2, per-lane global scratch) while the
//     children hold <= TL vertices in total;
//   * children above TL vertices: the node is posted to the CTA and updated by
//     a whole warp (pwl_heavy.cuh node_update_block, tier 3), any warp of the
//     CTA serving posted nodes while it waits (work sharing: the ~16 heavy
//     nodes of a level of a call buyer are the parallelism of that level).
// Carry records hold C inline vertices or an offset into the strip's carry
// arena.  Any capacity overflow aborts the item; the host re-runs it with 4x
// arenas (amtc_capi.cu), never truncating a function.
#include <cuda_runtime.h>

#include "amtc_internal.cuh"
#include "amtc_option.cuh"
#include "amtc_root.cuh"
#include "pwl_device.cuh"
#include "pwl_heavy.cuh"
#include "pwl_lane.cuh"

namespace amtc {

// shape (developer sweeps: -DAMTC_F_WARPS=... etc.)
#ifndef AMTC_F_C
#define AMTC_F_C 6
#endif
#ifndef AMTC_F_B
#define AMTC_F_B 10
#endif
#ifndef AMTC_F_WARPS
#define AMTC_F_WARPS 12
#endif
// developer instrumentation (-DAMTC_F_PROF=1): per-warp clock64 accumulators
// summed into g_fprof at kernel end, read by amtc_debug_full_profile
#ifndef AMTC_F_PROF
#define AMTC_F_PROF 0
#endif
__device__ unsigned long long g_fprof[8];
#if AMTC_F_PROF
#define FPROF_DECL unsigned long long fp_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; const long long fp_start = clock64();
#define FPROF_T(v) const long long v = clock64();
#define FPROF_ADD(i, x) fp_[i] += (unsigned long long)(x);
#else
#define FPROF_DECL
#define FPROF_T(v)
#define FPROF_ADD(i, x)
#endif
constexpr int FW = 34;  // strip matrix columns: 32 lanes + 2 carry columns (by level parity)
constexpr int F_BG = 256;  // vertices of each of a lane's two global scratch buffers (tier 2)
constexpr unsigned FFULL = 0xffffffffu;

template <int C>
struct FCarry {  // one level of a strip's carry column: [0] left slope, [1] (n, arena offset | -1), vertices
    double d[2 + 3 * C];
};

struct FMail {  // a heavy node posted to the CTA
    const Vtx* up;
    const Vtx* dp;
    double usl, dsl, lo, hi, ux, uf;
    int un, dn;
    short ustr, dstr;
    int res_err, res_n, res_off;
};

template <int C, int B>
struct FullSmem {
    Vtx row[C * FW];   // vertex i of column c at row[i * FW + c]
    Vtx scr[B * 32];   // pass-1 scratch (A) of lane l: scr[i * 32 + l]
    double csl[2];     // carry columns 32 / 33: left-tail slope, count, carry-arena offset (-1: inline)
    int cn[2], coff[2];
    int rcnt[2];       // row arena bump counters (by level parity)
    int ccnt;          // carry arena bump counter (this strip)
    int zcnt;          // scratch counter of the fallback heavy update
    heavy::HWin hw;    // merge windows of the tier-3 update this warp serves
    FMail mail[32];    // this warp's posted heavy nodes (one per lane)
    Vtx* h_arena;      // where their results go (this warp's next row arena) ...
    int* h_counter;    // ... and its bump counter
    int h_acap, h_seller;
    unsigned post;     // posted, not yet claimed heavy lanes
    int done;          // posted, not yet completed
};

struct FCtaHdr {
    int active;  // warps still working on items
    int posted;  // heavy nodes posted and not yet claimed
    int pad[2];
};

// per-warp global workspace layout (bytes), capacities in vertices
struct FullLayout {
    size_t rec, rec_ps;          // carry records (2 strip parities x (N+2) levels)
    size_t carena, carena_ps;    // carry arena (per strip parity)
    size_t rarena, rarena_ps;    // row arena (per level parity)
    size_t lscr, hscr, zbuf;     // tier-2 lane scratch (32 x 2 x F_BG), tier-3 scratch and output
    size_t total;
    int carena_cap, rarena_cap, hscr_cap, zbuf_cap, TL;
};

struct FullLaunch {
    BatchPtrs in;
    int N;
    Quote* out;
    const int* items;
    const int* item_lo;
    const int* n_items;
    int* work_counter;
    int* ovf_items;
    int* ovf_count;
    unsigned long long* vertex_sum;
    char* ws;
    FullLayout lay;
    double* hedge;
};

__host__ __device__ inline size_t f_align(size_t b) { return (b + 255) & ~(size_t)255; }

static FullLayout full_layout(int N, int level) {
    int rarena, carena, hscr, zbuf, tl;
    strip_tc_caps(N, level, rarena, carena, hscr, zbuf, tl);
    FullLayout L;
    L.rarena_cap = rarena;
    L.carena_cap = carena;
    L.hscr_cap = hscr;
    L.zbuf_cap = zbuf;
    L.TL = tl;
    size_t p = 0;
    auto take = [&](size_t bytes) { size_t q = p; p += f_align(bytes); return q; };
    L.rec_ps = f_align(sizeof(FCarry<AMTC_F_C>) * ((size_t)N + 2));
    L.rec = take(2 * L.rec_ps);
    L.carena_ps = f_align(sizeof(Vtx) * (size_t)L.carena_cap);
    L.carena = take(2 * L.carena_ps);
    L.rarena_ps = f_align(sizeof(Vtx) * (size_t)L.rarena_cap);
    L.rarena = take(2 * L.rarena_ps);
    L.lscr = take(sizeof(Vtx) * 32 * 2 * F_BG);
    L.hscr = take(sizeof(Vtx) * (size_t)L.hscr_cap);
    L.zbuf = take(sizeof(Vtx) * (size_t)L.zbuf_cap);
    L.total = p;
    return L;
}

// warp copy of n vertices between non-overlapping global buffers, eight loads
// in flight per lane before the stores
__device__ __forceinline__ void f_copy_vtx(Vtx* dst, const Vtx* src, int n, int lane) {
    const double* __restrict__ sp = reinterpret_cast<const double*>(src);
    double* __restrict__ dp = reinterpret_cast<double*>(dst);
    const int m = 3 * n;
    int i = lane;
    for (; i + 224 < m; i += 256) {
        double r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = sp[i + 32 * q];
#pragma unroll
        for (int q = 0; q < 8; ++q) dp[i + 32 * q] = r[q];
    }
    for (; i < m; i += 32) dp[i] = sp[i];
}

// tier 3 work sharing: claim one posted heavy node of any warp of the CTA
// (starting with this one), update it with the whole warp into this warp's
// scratch and copy it into the owner's row arena.  Returns true if it served.
template <int C, int B, int WARPS>
__device__ __noinline__ bool f_serve_one(FCtaHdr& H, FullSmem<C, B>* all, int me, Vtx* hscr, int hcap, Vtx* zbuf,
                                         int zcap, int lane) {
    unsigned pw = 0;
    if (lane < WARPS) pw = *(volatile unsigned*)&all[(me + lane) % WARPS].post;
    unsigned cand = __ballot_sync(FFULL, pw != 0);
    int owner = -1, ol = -1;
    while (cand && owner < 0) {
        const int c = __ffs(cand) - 1;
        cand &= cand - 1;
        const int w = (me + c) % WARPS;
        int got = -1;
        if (lane == 0) {
            unsigned cur = *(volatile unsigned*)&all[w].post;
            while (cur) {
                const unsigned bit = cur & (0u - cur);
                const unsigned old = atomicAnd(&all[w].post, ~bit);
                if (old & bit) {
                    got = __ffs(bit) - 1;
                    atomicSub(&H.posted, 1);
                    break;
                }
                cur = old & ~bit;
            }
        }
        got = __shfl_sync(FFULL, got, 0);
        if (got >= 0) { owner = w; ol = got; }
    }
    if (owner < 0) return false;
    FullSmem<C, B>& O = all[owner];
    const FMail& M = O.mail[ol];
    const Fn U = make_fn(M.up, M.un, M.usl, M.ustr), D = make_fn(M.dp, M.dn, M.dsl, M.dstr);
    const bool seller = O.h_seller != 0;
    int nZ = 0;
    int e = heavy::node_update_block(U, D, M.lo, M.hi, M.ux, M.uf, seller, &all[me].hw, hscr, hcap, zbuf, zcap, nZ,
                                     lane);
    if (e == heavy::DEV_FALLBACK) {  // rare shapes: the lane-contiguous update
        if (lane == 0) all[me].zcnt = 0;
        __syncwarp();
        int zoff = 0;
        e = heavy::node_update(U, D, M.lo, M.hi, M.ux, M.uf, seller, hscr, hcap, zbuf, &all[me].zcnt, zcap, zoff, nZ,
                               lane);
    }
    int off = 0;
    if (!e) {
        if (lane == 0) off = atomicAdd(O.h_counter, nZ);
        off = __shfl_sync(FFULL, off, 0);
        if (off + nZ > O.h_acap) e = DEV_OVERFLOW;
        else
            f_copy_vtx(O.h_arena + off, zbuf, nZ, lane);
    }
    __syncwarp();
    if (lane == 0) {
        O.mail[ol].res_err = e;
        O.mail[ol].res_n = nZ;
        O.mail[ol].res_off = off;
        __threadfence_block();
        atomicSub(&O.done, 1);
    }
    __syncwarp();
    return true;
}

// tier 2 (out of line: keeps the strip loop's registers for the common case):
// the node update by one lane with runtime strides, A in lg0 and z in lg1 (the
// lane's global scratch); returns the device status, z's count and left slope
static __device__ __noinline__ int f_tier2(const Fn U, const Fn D, double lo, double hi, double ux, double uf,
                                           bool seller, Vtx* lg0, Vtx* lg1, int& m, double& sl) {
    int nA = 0;
    double slA = lo;
    int e = lane_pass1(U, D, lo, lg0, F_BG, 1, nA, slA);
    if (e) return e;
    EmitT<1> G;
    G.out = lg1;
    G.cap = F_BG;
    G.stride = 1;
    e = lane_pass2<1>(make_fn_s<1>(lg0 + (F_BG - nA), nA, slA), lo, hi, ux, uf, seller, G);
    m = G.m;
    sl = G.sl;
    return e;
}
// pass 2 of a node whose A sits in the shared scratch but whose z outgrew the
// strip matrix: z into lg1
static __device__ __noinline__ int f_pass2_wide(const Vtx* A, int nA, double slA, double lo, double hi, double ux,
                                                double uf, bool seller, Vtx* lg1, int& m, double& sl) {
    EmitT<1> G;
    G.out = lg1;
    G.cap = F_BG;
    G.stride = 1;
    const int e = lane_pass2<1>(make_fn_s<32>(A, nA, slA), lo, hi, ux, uf, seller, G);
    m = G.m;
    sl = G.sl;
    return e;
}

template <int C, int B, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) full_kernel(const __grid_constant__ FullLaunch L) {
    static_assert(2 + 3 * C <= 32, "one lane per double of a carry record");
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    FCtaHdr& H = *reinterpret_cast<FCtaHdr*>(smem_raw);
    FullSmem<C, B>* const all = reinterpret_cast<FullSmem<C, B>*>(smem_raw + sizeof(FCtaHdr));
    FullSmem<C, B>& S = all[wib];
    const int N = L.N;
    char* const wb = L.ws + (size_t)(blockIdx.x * WARPS + wib) * L.lay.total;
    Vtx* const hscr = reinterpret_cast<Vtx*>(wb + L.lay.hscr);
    Vtx* const zbuf = reinterpret_cast<Vtx*>(wb + L.lay.zbuf);
    Vtx* const lg0 = reinterpret_cast<Vtx*>(wb + L.lay.lscr) + (size_t)lane * 2 * F_BG;  // pass-1 output (A)
    Vtx* const lg1 = lg0 + F_BG;                                                           // pass-2 output (z)
    if (threadIdx.x == 0) {
        H.active = WARPS;
        H.posted = 0;
    }
    if (lane == 0) {
        S.post = 0u;
        S.done = 0;
    }
    __syncthreads();
    FPROF_DECL
    const int item_lo = L.item_lo ? *L.item_lo : 0;
    for (;;) {
        int it = 0;
        if (lane == 0) it = item_lo + atomicAdd(L.work_counter, 1);
        it = __shfl_sync(FFULL, it, 0);
        if (it >= *L.n_items) break;
        const int code = L.items[it];
        const int64_t opt = code >> 1;
        const bool seller = (code & 1) == 0;
        OptionConsts oc;
        if (validate_option(L.in, opt, N, true, oc) != STATUS_OK) continue;  // status set by prepare
        const double kp = 1.0 + oc.k, km = 1.0 - oc.k;  // ask / bid factors
        const double e_h = exp(-oc.h), e_r = exp(oc.rho);
        const bool euro = (oc.flags & FLAG_EUROPEAN) != 0;
        int err = DEV_OK;
        int maxn = 1;
        unsigned long long vsum = 0;
        int my_n = 1, my_off = -1;
        double my_sl = 0.0;
        int cur = 0;  // row arena of the current input level

        for (int s = N / 32; s >= 0; --s) {
            const int j0 = 32 * s, j = j0 + lane;
            FCarry<C>* const rout = reinterpret_cast<FCarry<C>*>(wb + L.lay.rec + (size_t)(s & 1) * L.lay.rec_ps);
            const FCarry<C>* const rin =
                reinterpret_cast<const FCarry<C>*>(wb + L.lay.rec + (size_t)((s + 1) & 1) * L.lay.rec_ps);
            Vtx* const aout = reinterpret_cast<Vtx*>(wb + L.lay.carena + (size_t)(s & 1) * L.lay.carena_ps);
            const Vtx* const ain =
                reinterpret_cast<const Vtx*>(wb + L.lay.carena + (size_t)((s + 1) & 1) * L.lay.carena_ps);
            // a2: leaves t = N+1, payoff (0,0): z = y^- S^a - y^+ S^b, discounted (A11)
            {
                const double dN1 = exp(-oc.rho * (double)(N + 1));
                const double Sd = oc.S0 * exp(oc.h * (double)((N + 1) - 2 * j)) * dN1;
                S.row[lane] = Vtx{0.0, 0.0, -km * Sd};
                my_n = 1;
                my_off = -1;
                my_sl = -kp * Sd;
                if (lane == 31) {  // lane 31's down child at t = N: the leaf (N+1, j+1)
                    const double Sd1 = oc.S0 * exp(oc.h * (double)((N + 1) - 2 * (j + 1))) * dN1;
                    const int par = (N + 1) & 1;
                    S.row[32 + par] = Vtx{0.0, 0.0, -km * Sd1};
                    S.cn[par] = 1;
                    S.coff[par] = -1;
                    S.csl[par] = -kp * Sd1;
                }
                if (lane == 0) {
                    S.rcnt[0] = 0;
                    S.rcnt[1] = 0;
                    S.ccnt = 0;
                }
            }
            double Sq = oc.S0 * exp(oc.h * (double)(N - 2 * j));  // S_{t,j}, one multiply per level
            double disc = exp(-oc.rho * (double)N);                // r^-t
            const bool has_right = s < N / 32;
            double pre = 0.0;  // this lane's double of the next level's carry record
            const int t_end = max(j0, 1);
            for (int t = N; t >= t_end; --t) {
                const int nxt = cur ^ 1;
                const int par1 = (t + 1) & 1;  // carry column holding level t+1
                // carry of level t+1 (loaded during level t+1) -> column 32 + par1
                if (t < N && has_right && t + 1 >= j0 + 32) {
                    if (lane == 0) S.csl[par1] = pre;
                    else if (lane == 1) {
                        S.cn[par1] = __double2loint(pre);
                        S.coff[par1] = __double2hiint(pre);
                    } else if (lane < 2 + 3 * C) {
                        const int q = lane - 2;
                        (&S.row[(q / 3) * FW + 32 + par1].x)[q % 3] = pre;
                    }
                }
                // prefetch the record of level t (lane 31's down child at level t-1)
                if (has_right && t >= j0 + 32 && lane < 2 + 3 * C) pre = rin[t].d[lane];
                __syncwarp();
                if (*(volatile int*)&H.posted > 0) {
                    FPROF_T(t0)
                    const bool sv = f_serve_one<C, B, WARPS>(H, all, wib, hscr, L.lay.hscr_cap, zbuf, L.lay.zbuf_cap, lane);
                    FPROF_T(t1)
                    FPROF_ADD(0, t1 - t0) FPROF_ADD(4, sv)
                }
                const bool active = j <= t;
                // children: up = own previous, down = lane+1's previous / the carry column
                int dn = __shfl_down_sync(FFULL, my_n, 1);
                int doff = __shfl_down_sync(FFULL, my_off, 1);
                double dsl = __shfl_down_sync(FFULL, my_sl, 1);
                const int dcol = lane < 31 ? lane + 1 : 32 + par1;
                const Vtx* const rcur = reinterpret_cast<const Vtx*>(wb + L.lay.rarena + (size_t)cur * L.lay.rarena_ps);
                const Vtx* dbase = rcur;
                if (lane == 31) {
                    dn = S.cn[par1];
                    dsl = S.csl[par1];
                    doff = S.coff[par1];
                    dbase = ain;
                }
                // node constants: quotes (discounted), exercise function u_t (P:96 / P:133)
                const double Sd = Sq * disc;
                const double lo = -kp * Sd, hi = -km * Sd;
                double xi, zeta;
                option_payoff(oc, Sq, xi, zeta);
                const double ux = seller ? zeta : -zeta;
                double uf = (seller ? xi : -xi) * disc;
                if (euro && t < N) uf = seller ? -1e300 : 1e300;  // NEXT #3: no exercise before N
                const Fn Ug = my_off < 0 ? make_fn(&S.row[lane], my_n, my_sl, FW) : make_fn(rcur + my_off, my_n, my_sl, 1);
                const Fn Dg = doff < 0 ? make_fn(&S.row[dcol], dn, dsl, FW) : make_fn(dbase + doff, dn, dsl, 1);
                int e = DEV_OK, nA = 0, m2 = 0;
                double slA = lo, sl2 = lo;
                int where = 0;  // 1: A in the shared scratch; 2: z in the lane's global scratch lg1
                bool heavy = false;
                if (active) {
                    if (my_off < 0 && doff < 0) {  // both children in the strip matrix: compile-time strides
                        const FnT<FW> U = make_fn_s<FW>(&S.row[lane], my_n, my_sl);
                        const FnT<FW> D = make_fn_s<FW>(&S.row[dcol], dn, dsl);
                        e = lane_pass1<32>(U, D, lo, &S.scr[lane], B, 32, nA, slA);
                        where = 1;
                        if (e == DEV_OVERFLOW) where = 2;
                    } else if (my_n + dn > L.lay.TL) {
                        heavy = true;
                    } else {
                        where = 2;
                    }
                    if (where == 2) {
                        FPROF_T(t0)
                        e = f_tier2(Ug, Dg, lo, hi, ux, uf, seller, lg0, lg1, m2, sl2);
                        FPROF_T(t1)
                        FPROF_ADD(6, t1 - t0)
                        if (e == DEV_OVERFLOW) {  // too big for a lane: the warp takes the node
                            e = DEV_OK;
                            heavy = true;
                            where = 0;
                        }
                    }
                }
                // tier 3: post this level's heavy nodes to the CTA and serve until they are done
                int h_n = 0, h_off = 0;
                if (const unsigned hmask = __ballot_sync(FFULL, heavy)) {
                    if (heavy) {
                        FMail& m = S.mail[lane];
                        m.up = Ug.p; m.un = Ug.n; m.usl = Ug.sl; m.ustr = (short)Ug.stride;
                        m.dp = Dg.p; m.dn = Dg.n; m.dsl = Dg.sl; m.dstr = (short)Dg.stride;
                        m.lo = lo; m.hi = hi; m.ux = ux; m.uf = uf;
                    }
                    if (lane == 0) {
                        S.h_arena = reinterpret_cast<Vtx*>(wb + L.lay.rarena + (size_t)nxt * L.lay.rarena_ps);
                        S.h_counter = &S.rcnt[nxt];
                        S.h_acap = L.lay.rarena_cap;
                        S.h_seller = seller ? 1 : 0;
                        S.done = __popc(hmask);
                    }
                    __syncwarp();
                    __threadfence_block();
                    if (lane == 0) {
                        atomicAdd(&H.posted, __popc(hmask));
                        atomicOr(&S.post, hmask);
                    }
                    __syncwarp();
                    FPROF_T(w0)
                    while (*(volatile int*)&S.done > 0) {
                        FPROF_T(t0)
                        const bool sv = *(volatile int*)&H.posted > 0 &&
                            f_serve_one<C, B, WARPS>(H, all, wib, hscr, L.lay.hscr_cap, zbuf, L.lay.zbuf_cap, lane);
                        FPROF_T(t1)
                        if (sv) { FPROF_ADD(0, t1 - t0) FPROF_ADD(4, 1) FPROF_ADD(1, t0 - t1) }
                        else __nanosleep(64);
                    }
                    FPROF_T(w1)
                    FPROF_ADD(1, w1 - w0) FPROF_ADD(5, 1)
                    __threadfence_block();
                    if (heavy) {
                        const volatile FMail& m = S.mail[lane];
                        e |= m.res_err;
                        h_n = m.res_n;
                        h_off = m.res_off;
                    }
                }
                __syncwarp();  // every lane has read its children: the row may be overwritten
                if (active) {
                    if (heavy) {
                        my_n = h_n;
                        my_off = h_off;
                        my_sl = lo;
                    } else if (e == DEV_OK) {
                        if (where == 1) {  // z into the strip matrix when it fits
                            EmitT<FW> E;
                            E.out = &S.row[lane];
                            E.cap = C;
                            E.stride = FW;
                            e = lane_pass2<FW>(make_fn_s<32>(&S.scr[lane] + (B - nA) * 32, nA, slA), lo, hi, ux, uf,
                                               seller, E);
                            my_n = E.m;
                            my_sl = E.sl;
                            my_off = -1;
                            if (e == DEV_OVERFLOW) {
                                e = f_pass2_wide(&S.scr[lane] + (B - nA) * 32, nA, slA, lo, hi, ux, uf, seller, lg1, m2,
                                                 sl2);
                                where = 2;
                            }
                        }
                        if (where == 2 && e == DEV_OK) {  // z in lg1: into the strip matrix or the row arena
                            my_n = m2;
                            my_sl = sl2;
                            if (m2 <= C) {
                                for (int i = 0; i < m2; ++i) S.row[i * FW + lane] = lg1[i];
                                my_off = -1;
                            } else {
                                const int off = atomicAdd(&S.rcnt[nxt], m2);
                                if (off + m2 > L.lay.rarena_cap) {
                                    e = DEV_OVERFLOW;
                                } else {
                                    Vtx* const dst =
                                        reinterpret_cast<Vtx*>(wb + L.lay.rarena + (size_t)nxt * L.lay.rarena_ps) + off;
                                    for (int i = 0; i < m2; ++i) dst[i] = lg1[i];
                                    my_off = off;
                                }
                            }
                        }
                    }
                    err |= e;
                    maxn = max(maxn, my_n);
                    vsum += (unsigned long long)my_n;
                }
                __syncwarp();
                // carry out: node (t, j0), read by strip s-1's lane 31 at level t-1
                if (s > 0) {
                    const int c_n = __shfl_sync(FFULL, my_n, 0);
                    const int c_off = __shfl_sync(FFULL, my_off, 0);
                    const double c_sl = __shfl_sync(FFULL, my_sl, 0);
                    double* const rec = rout[t].d;
                    int base = -1;
                    if (c_off >= 0) {  // a wide function: copy it into this strip's carry arena
                        if (lane == 0) base = atomicAdd(&S.ccnt, c_n);
                        base = __shfl_sync(FFULL, base, 0);
                        if (base + c_n > L.lay.carena_cap) {
                            err |= DEV_OVERFLOW;
                            base = 0;
                        } else {
                            const Vtx* const src =
                                reinterpret_cast<const Vtx*>(wb + L.lay.rarena + (size_t)nxt * L.lay.rarena_ps) + c_off;
                            f_copy_vtx(aout + base, src, c_n, lane);
                        }
                    }
                    if (lane == 0) rec[0] = c_sl;
                    else if (lane == 1) rec[1] = __hiloint2double(base, c_n);
                    else if (c_off < 0 && lane < 2 + 3 * min(c_n, C)) {
                        const int q = lane - 2;
                        rec[lane] = (&S.row[(q / 3) * FW].x)[q % 3];
                    }
                }
                if (lane == 0) S.rcnt[cur] = 0;  // level t+1's row arena is dead
                cur = nxt;
                Sq *= e_h;
                disc *= e_r;
                err = __reduce_or_sync(FFULL, err);
                if (err) break;
                __syncwarp();
            }
            if (err) break;
            if (s == 0) {
                const Vtx* const rc = reinterpret_cast<const Vtx*>(wb + L.lay.rarena + (size_t)cur * L.lay.rarena_ps);
                const Fn mine = my_off < 0 ? make_fn(&S.row[lane], my_n, my_sl, FW) : make_fn(rc + my_off, my_n, my_sl, 1);
                err |= tc_root(mine, oc, seller, &L.out[opt],
                               L.hedge ? &L.hedge[2 * opt + (seller ? 0 : 1)] : nullptr, lane);
            }
            __syncwarp();
        }
        // per-item bookkeeping
        err = __reduce_or_sync(FFULL, err);
        maxn = __reduce_max_sync(FFULL, maxn);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(FFULL, vsum, o);
        if (lane == 0) {
            atomicAdd(L.vertex_sum, vsum);
            if (err & DEV_OVERFLOW) {  // re-run with larger arenas
                const int q = atomicAdd(L.ovf_count, 1);
                L.ovf_items[q] = code;
            } else if (err & DEV_UNBOUNDED) {
                atomicMax(&L.out[opt].status, STATUS_EUNBOUNDED);
            }
            atomicMax(&L.out[opt].max_bp, maxn);
        }
        __syncwarp();
    }
    // no items left: serve the CTA's remaining heavy nodes until every warp is done
    if (lane == 0) atomicSub(&H.active, 1);
    __syncwarp();
    FPROF_T(e0)
    unsigned nap = 256;
    while (*(volatile int*)&H.active > 0) {
        FPROF_T(t0)
        if (*(volatile int*)&H.posted > 0 &&
            f_serve_one<C, B, WARPS>(H, all, wib, hscr, L.lay.hscr_cap, zbuf, L.lay.zbuf_cap, lane)) {
            FPROF_T(t1)
            FPROF_ADD(0, t1 - t0) FPROF_ADD(4, 1) FPROF_ADD(2, t0 - t1)
            nap = 256;
        } else {
            __nanosleep(nap);
            nap = min(nap * 2, 32768u);
        }
    }
#if AMTC_F_PROF
    const long long fp_end = clock64();
    fp_[2] += (unsigned long long)(fp_end - e0);
    fp_[3] += (unsigned long long)(fp_end - fp_start);
    if (lane == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(&g_fprof[i], fp_[i]);
#endif
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
constexpr int F_C = AMTC_F_C, F_B = AMTC_F_B, F_WARPS = AMTC_F_WARPS;
#define FULL_KERNEL full_kernel<F_C, F_B, F_WARPS>
constexpr size_t F_SMEM = sizeof(FCtaHdr) + sizeof(FullSmem<F_C, F_B>) * F_WARPS;

static int full_set_smem() {
    static int done = 0;
    if (!done) {
        if (cudaFuncSetAttribute(FULL_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F_SMEM) !=
            cudaSuccess)
            return STATUS_ECUDA;
        done = 1;
    }
    return STATUS_OK;
}

size_t full_ws_bytes_per_warp(int N, int level) { return full_layout(N, level).total; }
int full_warps_per_cta() { return F_WARPS; }
int full_ctas_per_sm() {
    int b = 0;
    if (full_set_smem() != STATUS_OK) return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, FULL_KERNEL, F_WARPS * 32, F_SMEM);
    return b;
}

int full_profile(unsigned long long out[8], int reset) {
    if (cudaMemcpyFromSymbol(out, g_fprof, sizeof(unsigned long long) * 8) != cudaSuccess) return STATUS_ECUDA;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (cudaMemcpyToSymbol(g_fprof, z, sizeof(z)) != cudaSuccess) return STATUS_ECUDA;
    }
    return AMTC_F_PROF ? STATUS_OK : STATUS_EINVAL;
}

int full_launch(const StripLaunchArgs& a, cudaStream_t s) {
    FullLaunch L;
    L.in = a.in;
    L.N = a.N;
    L.out = a.out;
    L.items = a.items;
    L.item_lo = a.item_lo;
    L.n_items = a.n_items;
    L.work_counter = a.work_counter;
    L.ovf_items = a.ovf_items;
    L.ovf_count = a.ovf_count;
    L.vertex_sum = a.vertex_sum;
    L.ws = a.ws;
    L.lay = full_layout(a.N, a.level);
    L.hedge = a.hedge;
    if (L.lay.total != a.ws_stride) return STATUS_EINVAL;
    if (full_set_smem() != STATUS_OK) return STATUS_ECUDA;
    FULL_KERNEL<<<a.ctas, F_WARPS * 32, F_SMEM, s>>>(L);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STATUS_OK : STATUS_ECUDA;
}

}  // namespace amtc
