// amtc_strip.cu -- the batched transaction-cost solver: one warp per work item
// (option, party), the recombining tree swept in vertical strips.
//
// Recursion (Sec. 3; tree of Sec. 4.1): node (t, j)
// needs only its children (t+1, j) and (t+1, j+1), so the dependency cone of a
// node points to the RIGHT (larger j), as the paper's region-B argument notes
// (P:164-166).  The warp therefore covers the triangle in strips of 32 columns,
// right to left:
//
//   strip s owns columns j = 32 s + lane; it sweeps levels t = N .. max(32 s, 1)
//   (lane active iff j <= t).  Lane l's up child (t+1, j) is its own previous
//   result; the down child (t+1, j+1) is lane l+1's previous result, and for
//   lane 31 the column 32 (s+1) of the strip to the right -- the "carry"
//   column, written by that strip's lane 0 at every level (one function per
//   level, in global memory: the only per-level traffic that leaves the SM).
//   The leaves (t = N+1, payoff (0,0)) are analytic.
//
// This replaces the paper's p-thread block/region rounds (Alg. 1):
// the GPU analogue of its region-B dependency is the carry column; there are
// no barriers beyond __syncwarp, and no level is ever materialised in HBM.
//
// Node functions: a function is a vertex list
// (x, f, s_right) with its left-tail slope carried alongside (pwl_device.cuh);
// every function is stored discounted to t = 0 (z_t / r^t), so the paper's
// w_t / r is a plain max.  Storage:
//   * row slots: C vertices per lane, in shared memory, lane-interleaved
//     (vertex i of lane l at row[i * 32 + l]: conflict-free for any mix of i);
//   * functions with more than C vertices live in a per-warp global "row
//     arena" (ping-pong by level parity) -- the heavy "sawtooth" of the buyer
//     of calls / bull spreads;
//   * node-update scratch: B vertices x 2 buffers per lane in shared memory;
//     a node that outgrows it re-runs with per-lane global scratch (tier 2);
//   * nodes whose children hold more than TL vertices in total are updated by
//     the whole warp cooperatively (pwl_heavy.cuh, tier 3).
// Any capacity overflow aborts the item; the host re-runs it with larger
// arenas (amtc_capi.cu), never truncating a function.
#include <cuda_runtime.h>

#include <algorithm>

#include "amtc_internal.cuh"
#include "amtc_option.cuh"
#include "pwl_device.cuh"
#include "pwl_heavy.cuh"
#include "pwl_lane.cuh"
#include "amtc_root.cuh"

namespace amtc {

constexpr int SW = 32;  // strip width = lanes per warp

// per-warp global workspace: byte offsets of its regions (the second copy of
// a ping-pong pair sits at offset + *_ps); computed once on the host
struct StripLayout {
    size_t epow, dpow;          // 2N+3 / N+2 doubles: e^{h (i-(N+1))}, e^{-rho t}
    size_t chdr, csl, cv;       // carry column: header (n, arena offset | -1), left slope, C inline vertices
    size_t carena, rarena;      // carry arena (per strip parity), row arena (per level parity)
    size_t lscr, hscr, zbuf;    // tier-2 lane scratch (32 x 2 x BG), tier-3 warp scratch, tier-3 output
    size_t chdr_ps, csl_ps, cv_ps, carena_ps, rarena_ps;
    size_t total;
};

struct StripCaps {
    int C, B, BG, TL;
    int carena_cap, rarena_cap, hscr_cap, zbuf_cap;
};

__host__ __device__ inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static StripLayout strip_layout(int N, const StripCaps& c) {
    StripLayout L;
    const size_t nn = (size_t)N + 2;
    size_t p = 0;
    auto take = [&](size_t bytes) { size_t q = p; p += align256(bytes); return q; };
    L.epow = take(sizeof(double) * (2 * (size_t)N + 3));
    L.dpow = take(sizeof(double) * nn);
    L.chdr_ps = align256(sizeof(int2) * nn);
    L.chdr = take(2 * L.chdr_ps);
    L.csl_ps = align256(sizeof(double) * nn);
    L.csl = take(2 * L.csl_ps);
    L.cv_ps = align256(sizeof(Vtx) * nn * c.C);
    L.cv = take(2 * L.cv_ps);
    L.carena_ps = align256(sizeof(Vtx) * (size_t)c.carena_cap);
    L.carena = take(2 * L.carena_ps);
    L.rarena_ps = align256(sizeof(Vtx) * (size_t)c.rarena_cap);
    L.rarena = take(2 * L.rarena_ps);
    L.lscr = take(sizeof(Vtx) * (size_t)SW * 2 * c.BG);
    L.hscr = take(sizeof(Vtx) * (size_t)c.hscr_cap);
    L.zbuf = take(sizeof(Vtx) * (size_t)c.zbuf_cap);
    L.total = p;
    return L;
}

// a heavy node posted by one lane for the CTA's warps (tier 3 work sharing)
struct HMail {
    const Vtx* up;
    const Vtx* dp;
    double usl, dsl, lo, hi, ux, uf;
    int un, dn;
    short ustr, dstr;
    int res_err, res_n, res_off;
};

// per-warp shared memory
template <int C, int B>
struct StripSmemBase {
    Vtx row[C * SW];  // lane-interleaved slots: vertex i of lane l at row[i * 32 + l]
    Vtx s0[B * SW];   // lane-interleaved scratch of the node update (A of pass 1)
    Vtx leaf31;       // lane 31's down child at t = N (an analytic leaf)
    int rcnt[2];      // row arena bump counters
    int ccnt;         // carry arena bump counter (current strip)
    int zcnt;         // scratch counter of the fallback heavy update
};
// HEAVY = true: the tier-3 parts (the light-only kernel variant omits them)
template <int C, int B, bool HEAVY = true>
struct StripSmem : StripSmemBase<C, B> {
    heavy::HWin hw;   // merge windows of the tier-3 (heavy) node update
    HMail mail[SW];   // this warp's posted heavy nodes (one per lane)
    Vtx* h_arena;     // where their results go (this warp's next row arena) ...
    int* h_counter;   // ... and its bump counter
    int h_acap, h_seller;
    unsigned post;    // posted, not yet claimed heavy lanes
    int done;         // posted, not yet completed
};
template <int C, int B>
struct StripSmem<C, B, false> : StripSmemBase<C, B> {};

struct CtaHdr {
    int active;  // warps of this CTA still working on items
    int posted;  // heavy nodes posted and not yet claimed (cheap poll for helpers)
    int pad[2];
};

struct StripLaunch {
    BatchPtrs in;
    int N;
    Quote* out;
    const int* items;
    const int* n_items;
    int* work_counter;
    int* ovf_items;
    int* ovf_count;
    unsigned long long* vertex_sum;
    char* ws;
    StripCaps caps;
    StripLayout lay;
    // split mode (one tree's strips on different warps): 0 = off, else strips per tree
    int split_S;
    int* progress;          // per (tree, strip): lowest level whose carry is published
    char* carry;            // per (tree, strip): chdr | csl | cv, carry_stride bytes
    size_t carry_stride, c_csl, c_cv;
    Vtx* carena_split;      // per tree: carry arena, carena_split_cap vertices
    int* carena_cnt;        // per tree: its bump counter
    int carena_split_cap;
    const int* item_lo;     // device: first item index of this launch (nullptr: 0)
    // sharded single tree: strip peer_strip (and its carry arena / progress) is
    // owned by the next GPU, mapped here through CUDA IPC; -1: none
    int peer_strip;
    int sys_fence;          // publish progress with system-scope fences
    char* peer_carry;
    Vtx* peer_carena;
    int* peer_progress;
    double* hedge;          // optional: root hedge per (option, party) (2 n doubles)
};

#define WS(T, field, q) reinterpret_cast<T*>(wb + L.lay.field + (size_t)(q) * L.lay.field##_ps)
#define WS1(T, field) reinterpret_cast<T*>(wb + L.lay.field)

// carry-column pointers of strip s (out) or of the strip to its right (in),
// rebuilt at each use from the launch parameters instead of being kept live
// across the level loop (register pressure: the loop state spills otherwise)
struct CarryPtrs {
    int2* chdr;
    double* csl;
    Vtx* cv;
    Vtx* ca;
};
__device__ __forceinline__ CarryPtrs carry_ptrs(const StripLaunch& L, char* wb, int tree, int s, bool split,
                                                bool input) {
    CarryPtrs P;
    if (split) {
        const bool remote = input && s + 1 == L.peer_strip;
        const size_t si = (size_t)tree * L.split_S + s + (input ? 1 : 0);
        char* c = (remote ? L.peer_carry : L.carry) + si * L.carry_stride;
        P.chdr = reinterpret_cast<int2*>(c);
        P.csl = reinterpret_cast<double*>(c + L.c_csl);
        P.cv = reinterpret_cast<Vtx*>(c + L.c_cv);
        P.ca = (remote ? L.peer_carena : L.carena_split) + (size_t)tree * L.carena_split_cap;
    } else {
        const int q = (s & 1) ^ (input ? 1 : 0);
        P.chdr = reinterpret_cast<int2*>(wb + L.lay.chdr + (size_t)q * L.lay.chdr_ps);
        P.csl = reinterpret_cast<double*>(wb + L.lay.csl + (size_t)q * L.lay.csl_ps);
        P.cv = reinterpret_cast<Vtx*>(wb + L.lay.cv + (size_t)q * L.lay.cv_ps);
        P.ca = reinterpret_cast<Vtx*>(wb + L.lay.carena + (size_t)q * L.lay.carena_ps);
    }
    return P;
}

// copy n vertices between (possibly strided) locations, one lane
__device__ __forceinline__ void copy_fn(Vtx* dst, int dstride, const Vtx* src, int sstride, int n) {
    for (int i = 0; i < n; ++i) dst[i * dstride] = src[i * sstride];
}


constexpr unsigned FULL = 0xffffffffu;


// tier 3 (work sharing inside the CTA): a warp whose level has heavy nodes
// posts them (HMail per lane, bit mask `post`) and then serves posted nodes --
// its own or any other warp's -- until its own are done; every warp also
// serves one posted node per level of its own sweep, and warps without items
// serve until the CTA is idle.  A claimed node is updated by the whole warp
// (pwl_heavy.cuh) into the claimer's scratch and copied into the owner's row
// arena.  Returns true if a node was served.

// warp copy of n vertices between global buffers that never overlap, as 3n
// doubles with eight loads in flight per lane before the stores (the compiler
// cannot reorder a load above a store through possibly aliasing pointers, so a
// plain loop waits one memory latency per 32 vertices)
static_assert(sizeof(Vtx) == 3 * sizeof(double), "warp_copy_vtx copies vertices as doubles");
__device__ __forceinline__ void warp_copy_vtx(Vtx* dst, const Vtx* src, int n, int lane) {
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

template <int C, int B, int WARPS>
__device__ __noinline__ bool serve_one(CtaHdr& H, StripSmem<C, B, true>* all, int me, Vtx* hscr, int hcap, Vtx* zbuf,
                                       int zcap, int lane) {
    // candidate owner: the first warp (starting with this one) with posted nodes
    unsigned pw = 0;
    if (lane < WARPS) pw = *(volatile unsigned*)&all[(me + lane) % WARPS].post;
    unsigned cand = __ballot_sync(FULL, pw != 0);
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
        got = __shfl_sync(FULL, got, 0);
        if (got >= 0) { owner = w; ol = got; }
    }
    if (owner < 0) return false;
    StripSmem<C, B, true>& O = all[owner];
    const HMail& M = O.mail[ol];
    const Fn U = make_fn(M.up, M.un, M.usl, M.ustr), D = make_fn(M.dp, M.dn, M.dsl, M.dstr);
    const bool seller = O.h_seller != 0;
    int nZ = 0;
    // rolled scan loops for the fetch-bound 20-warp batch shape, unrolled ones for the
    // latency-bound 16-warp split shape (pwl_heavy.cuh, RL)
    constexpr bool RL = WARPS > 16 && heavy::RL_DEFAULT;
    int e = heavy::node_update_block<heavy::HWin*, RL>(U, D, M.lo, M.hi, M.ux, M.uf, seller, &all[me].hw, hscr, hcap, zbuf,
                                                       zcap, nZ, lane);
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
        off = __shfl_sync(FULL, off, 0);
        if (off + nZ > O.h_acap) e = DEV_OVERFLOW;
        else
            warp_copy_vtx(O.h_arena + off, zbuf, nZ, lane);
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

template <int C, int B, int WARPS, int MINB, bool HEAVY>
__global__ void __launch_bounds__(WARPS * 32, MINB) strip_kernel(const __grid_constant__ StripLaunch L) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    CtaHdr& H = *reinterpret_cast<CtaHdr*>(smem_raw);
    StripSmem<C, B, HEAVY>* const all = reinterpret_cast<StripSmem<C, B, HEAVY>*>(smem_raw + sizeof(CtaHdr));
    StripSmem<C, B, HEAVY>& S = all[wib];
    const int N = L.N;
    char* const wb = L.ws + (size_t)(blockIdx.x * WARPS + wib) * L.lay.total;
#define Epow WS1(double, epow)
#define Dpow WS1(double, dpow)
#define hscr WS1(Vtx, hscr)
#define zbuf WS1(Vtx, zbuf)
    if (threadIdx.x == 0) {
        H.active = WARPS;
        H.posted = 0;
    }
    if constexpr (HEAVY) {
        if (lane == 0) {
            S.post = 0u;
            S.done = 0;
        }
    }
    __syncthreads();

    const int item_lo = L.item_lo ? *L.item_lo : 0;
    const bool split = L.split_S > 0;
    // Whole-tree mode: each warp's FIRST item is dealt statically, in snake order
    // over the CTAs (warp w of CTA b takes queue position w G + b, or w G + G-1-b
    // for odd w); later items come from the atomic ticket counter.  The queue is
    // ordered heavy-first and the warps of a CTA start together, so with tickets
    // alone CTA 0 drew the 20 heaviest items of the batch, CTA 1 the next 20, ...
    // -- one SM then carried several times the mean load, which a batch of about
    // one item per warp (a multi-GPU slice) never evens out.  Split mode keeps
    // pure ticket order (strips must be claimed right to left).
    bool first_item = !split;
    for (;;) {
        int it = 0;
        if (first_item) {
            const int G = (int)gridDim.x, b = (int)blockIdx.x;
            it = item_lo + wib * G + ((wib & 1) ? G - 1 - b : b);
            first_item = false;
        } else {
            if (lane == 0) it = item_lo + (split ? 0 : (int)gridDim.x * WARPS) + atomicAdd(L.work_counter, 1);
            it = __shfl_sync(FULL, it, 0);
        }
        if (it >= *L.n_items) break;
        const int code = L.items[it];
        const int tree = split ? code / L.split_S : code;  // 2 option + party
        const int s_first = split ? code % L.split_S : N / SW, s_last = split ? s_first : 0;
        const int64_t opt = tree >> 1;
        const bool seller = (tree & 1) == 0;
        OptionConsts oc;
        if (validate_option(L.in, opt, N, true, oc) != STATUS_OK) continue;  // status set by prepare

        // a1: per-option tables: S_{t,j} = S0 e^{h (t-2j)}, r^-t = e^{-rho t}
        for (int i = lane; i < 2 * N + 3; i += 32) Epow[i] = exp(oc.h * (double)(i - (N + 1)));
        for (int t = lane; t < N + 2; t += 32) Dpow[t] = exp(-oc.rho * (double)t);
        __syncwarp();
        const double kp = 1.0 + oc.k, km = 1.0 - oc.k;  // ask / bid factors
        int err = DEV_OK;
        int maxn = 1;
        unsigned long long vsum = 0;

        for (int s = s_first; s >= s_last && !err; --s) {
            const int j0 = s * SW, j = j0 + lane;
            // split mode: progress counters of this strip and of the strip to its right
            volatile int* const prog_out = split ? L.progress + (size_t)tree * L.split_S + s : nullptr;
            // a2: leaves t = N+1, payoff (0,0): z = y^- S^a - y^+ S^b
            int my_n = 0, my_off = -1;
            double my_sl = 0.0;
            if (j <= N + 1) {
                const double Sd = oc.S0 * Epow[(N + 1) - 2 * j + (N + 1)] * Dpow[N + 1];
                Vtx& v = S.row[lane];
                v.x = 0.0;
                v.f = 0.0;
                v.s = -km * Sd;
                my_n = 1;
                my_sl = -kp * Sd;
                if (lane == 31 && j + 1 <= N + 1) {
                    const double Sd1 = oc.S0 * Epow[(N + 1) - 2 * (j + 1) + (N + 1)] * Dpow[N + 1];
                    S.leaf31.x = 0.0;
                    S.leaf31.f = 0.0;
                    S.leaf31.s = -km * Sd1;
                }
            }
            const double leaf31_sl = -kp * oc.S0 * Epow[max((N + 1) - 2 * (j + 1) + (N + 1), 0)] * Dpow[N + 1];
            if (lane == 0) {
                S.rcnt[0] = 0;
                S.rcnt[1] = 0;
                S.ccnt = 0;
            }
            __syncwarp();
            int cur = 0;
            for (int t = N; t >= max(j0, 1); --t) {
                const int nxt = cur ^ 1;
                const bool active = j <= t;
                // help: serve one heavy node posted by another warp of the CTA
                if constexpr (HEAVY) {
                    if (*(volatile int*)&H.posted > 0)
                        serve_one<C, B, WARPS>(H, all, wib, hscr, L.caps.hscr_cap, zbuf, L.caps.zbuf_cap, lane);
                }
                // children: up = own previous; down = lane+1's previous / carry / leaf
                const int dn = __shfl_down_sync(FULL, my_n, 1);
                const int doff = __shfl_down_sync(FULL, my_off, 1);
                const double dsl = __shfl_down_sync(FULL, my_sl, 1);
                Vtx* const rcur = WS(Vtx, rarena, cur);
                const Fn U = (my_off < 0) ? make_fn(&S.row[lane], my_n, my_sl, SW)
                                          : make_fn(rcur + my_off, my_n, my_sl, 1);
                Fn D;
                if (lane < 31) {
                    D = (doff < 0) ? make_fn(&S.row[lane + 1], dn, dsl, SW) : make_fn(rcur + doff, dn, dsl, 1);
                } else if (t == N) {
                    D = make_fn(&S.leaf31, 1, leaf31_sl, 1);  // the analytic leaf (N+1, j+1)
                } else if (active) {
                    int pv = 0;
                    if (split) {  // split mode: wait until strip s+1 has published level t+1
                        const bool remote = s + 1 == L.peer_strip;
                        volatile int* const prog_in =
                            (remote ? L.peer_progress : L.progress) + (size_t)tree * L.split_S + s + 1;
                        while ((pv = *prog_in) > t + 1) __nanosleep(32);
                        __threadfence();
                    }
                    if (pv < 0) {  // strip s+1 failed (capacity): finish with a dummy, re-run later
                        err |= DEV_OVERFLOW;
                        D = make_fn(&S.leaf31, 1, leaf31_sl, 1);
                    } else {
                        const CarryPtrs ci = carry_ptrs(L, wb, tree, s, split, true);
                        const volatile int* hp = reinterpret_cast<const volatile int*>(&ci.chdr[t + 1]);
                        const int2 h = make_int2(hp[0], hp[1]);
                        const double csl = *(volatile const double*)&ci.csl[t + 1];
                        D = (h.y < 0) ? make_fn(ci.cv + (size_t)(t + 1) * C, h.x, csl, 1)
                                      : make_fn(ci.ca + h.y, h.x, csl, 1);
                    }
                } else {
                    D = make_fn(&S.leaf31, 0, 0.0, 1);
                }
                // node constants: quotes (discounted), exercise function u_t (P:96 / P:133)
                const double S_ = oc.S0 * Epow[max(t - 2 * j + (N + 1), 0)];  // idle lanes: any index
                const double disc = Dpow[t];
                const double lo = -kp * S_ * disc, hi = -km * S_ * disc;
                double xi, zeta;
                option_payoff(oc, S_, xi, zeta);
                const double ux = seller ? zeta : -zeta;
                double uf = (seller ? xi : -xi) * disc;
                // European (NEXT #3): no exercise before N -- u moves out of reach, z = v
                if ((oc.flags & FLAG_EUROPEAN) && t < N) uf = seller ? -1e300 : 1e300;

                // tier 1 / tier 2: sequential update by this lane (pwl_lane.cuh).
                // Pass 1 reads the children and leaves A in the lane's scratch
                // (shared; the lane's global scratch when it outgrows B vertices).
                Vtx* const lg0 = WS1(Vtx, lscr) + (size_t)lane * 2 * L.caps.BG;
                int nA = 0;
                double slA = lo;
                int where = 0;  // A in: 1 = shared scratch, 2 = lane global scratch
                bool heavy = false;
                if (active) {
                    heavy = U.n + D.n > L.caps.TL;
                    // attempt 0: shared scratch; attempt 1: the lane's global scratch
                    for (int attempt = 0; attempt < 2 && !heavy; ++attempt) {
                        Vtx* const buf = attempt ? lg0 : &S.s0[lane];
                        const int e = lane_pass1(U, D, lo, buf, attempt ? L.caps.BG : B, attempt ? 1 : SW, nA, slA);
                        where = attempt + 1;
                        if (e != DEV_OVERFLOW) {
                            err |= e;
                            break;
                        }
                        if (attempt) heavy = true;  // too big for a lane: the warp takes it
                    }
                    if (heavy) where = 0;
                }
                // tier 3: post this level's heavy nodes to the CTA and serve until they are done
                int h_n = 0, h_off = 0;
                if constexpr (!HEAVY) {
                    if (heavy) err |= DEV_OVERFLOW;  // light-only kernel: re-run by the full kernel
                } else if (const unsigned hmask = __ballot_sync(FULL, heavy)) {
                    if (heavy) {
                        HMail& m = S.mail[lane];
                        m.up = U.p; m.un = U.n; m.usl = U.sl; m.ustr = (short)U.stride;
                        m.dp = D.p; m.dn = D.n; m.dsl = D.sl; m.dstr = (short)D.stride;
                        m.lo = lo; m.hi = hi; m.ux = ux; m.uf = uf;
                    }
                    if (lane == 0) {
                        S.h_arena = WS(Vtx, rarena, nxt);
                        S.h_counter = &S.rcnt[nxt];
                        S.h_acap = L.caps.rarena_cap;
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
                    while (*(volatile int*)&S.done > 0) {
                        if (*(volatile int*)&H.posted <= 0 ||
                            !serve_one<C, B, WARPS>(H, all, wib, hscr, L.caps.hscr_cap, zbuf, L.caps.zbuf_cap, lane))
                            __nanosleep(64);
                    }
                    __threadfence_block();
                    if (heavy) {
                        const volatile HMail& m = S.mail[lane];
                        err |= m.res_err;
                        h_n = m.res_n;
                        h_off = m.res_off;
                    }
                }
                __syncwarp();
                // pass 2 writes Z over the previous row, which is dead now (every
                // lane has read its children)
                if (active) {
                    if (heavy) {
                        my_n = h_n;
                        my_off = h_off;
                        my_sl = lo;
                    } else if (where && !err) {
                        const Fn A = (where == 1) ? make_fn(&S.s0[lane] + (size_t)(B - nA) * SW, nA, slA, SW)
                                                  : make_fn(lg0 + (L.caps.BG - nA), nA, slA, 1);
                        Vtx* const lg1 = lg0 + L.caps.BG;
                        Emit E;
                        int e = DEV_OK;
                        // attempt 0: straight into the row slot; 1: more than C vertices,
                        // via the lane scratch into the row arena
                        for (int attempt = 0; attempt < 2; ++attempt) {
                            E.out = attempt ? lg1 : &S.row[lane];
                            E.cap = attempt ? L.caps.BG : C;
                            E.stride = attempt ? 1 : SW;
                            e = lane_pass2(A, lo, hi, ux, uf, seller, E);
                            if (e != DEV_OVERFLOW) break;
                        }
                        my_off = -1;
                        if (!e && E.out == lg1) {
                            const int off = atomicAdd(&S.rcnt[nxt], E.m);
                            if (off + E.m > L.caps.rarena_cap) {
                                e = DEV_OVERFLOW;
                            } else {
                                copy_fn(WS(Vtx, rarena, nxt) + off, 1, lg1, 1, E.m);
                                my_off = off;
                            }
                        }
                        err |= e;
                        my_n = E.m;
                        my_sl = E.sl;
                    }
                    vsum += (unsigned long long)my_n;
                    maxn = max(maxn, my_n);
                }
                __syncwarp();
                // carry out: node (t, j0), read by the strip to the left (its lane 31 at level t-1)
                {
                    const int c_n = __shfl_sync(FULL, my_n, 0);
                    const int c_off = __shfl_sync(FULL, my_off, 0);
                    const CarryPtrs co = carry_ptrs(L, wb, tree, s, split, false);
                    if (lane == 0) co.csl[t] = my_sl;
                    if (c_off < 0) {
                        if (lane < c_n) co.cv[(size_t)t * C + lane] = S.row[lane * SW];
                        if (lane == 0) co.chdr[t] = make_int2(c_n, -1);
                    } else {
                        int base = 0;
                        if (lane == 0) base = atomicAdd(split ? &L.carena_cnt[tree] : &S.ccnt, c_n);
                        base = __shfl_sync(FULL, base, 0);
                        if (base + c_n > (split ? L.carena_split_cap : L.caps.carena_cap)) {
                            err |= DEV_OVERFLOW;
                        } else {
                            Vtx* const ca = co.ca + base;
                            const Vtx* const ra = WS(Vtx, rarena, nxt) + c_off;
                            warp_copy_vtx(ca, ra, c_n, lane);
                            if (lane == 0) co.chdr[t] = make_int2(c_n, base);
                        }
                    }
                    if (prog_out) {  // split mode: publish level t to strip s-1
                        if (L.sys_fence) __threadfence_system();  // the reader may be another GPU
                        else __threadfence();
                        __syncwarp();
                        if (lane == 0) *prog_out = t;
                    }
                }
                if (lane == 0) S.rcnt[cur] = 0;  // level t+1's arena is dead
                cur = nxt;
                err = __reduce_or_sync(FULL, err);
                if (err) break;
                __syncwarp();
            }
            __syncwarp();
            if (prog_out && err && lane == 0) {  // never leave strip s-1 waiting
                if (L.sys_fence) __threadfence_system();
                *prog_out = -1;
            }
            if (s == 0 && !err) {
                const Fn mine = (my_off < 0) ? make_fn(&S.row[lane], my_n, my_sl, SW)
                                             : make_fn(WS(Vtx, rarena, cur) + my_off, my_n, my_sl, 1);
                err |= tc_root(mine, oc, seller, &L.out[opt], L.hedge ? &L.hedge[2 * opt + (seller ? 0 : 1)] : nullptr,
                                  lane);
            }
        }
        // per-item bookkeeping
        err = __reduce_or_sync(FULL, err);
        maxn = __reduce_max_sync(FULL, maxn);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(FULL, vsum, o);
        if (lane == 0) {
            atomicAdd(L.vertex_sum, vsum);
            if (err & DEV_OVERFLOW) {
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
    if constexpr (HEAVY) {
        if (lane == 0) atomicSub(&H.active, 1);
        __syncwarp();
        unsigned nap = 256;  // exponential backoff while nothing is posted
        while (*(volatile int*)&H.active > 0) {
            if (*(volatile int*)&H.posted > 0 &&
                serve_one<C, B, WARPS>(H, all, wib, hscr, L.caps.hscr_cap, zbuf, L.caps.zbuf_cap, lane)) {
                nap = 256;
            } else {
                __nanosleep(nap);
                nap = min(nap * 2, 32768u);
            }
        }
    }
}

#undef Epow
#undef Dpow
#undef hscr
#undef zbuf

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// full kernel: one CTA of 20 warps per SM (the CTA is the work-sharing domain of
// tier 3), 3-vertex row slots and scratch (20 / 3: 7.48 s vs 20 / 4: 7.65 s per config-4 step with the
// rolled-scan heavy update; before it measured: 20 warps / 4 beat 16 / 6 by
// 2.5%, 12 / 6 and 8 / 6 lose 5-16%, 24 / 3 loses 2.5x).  Light kernel: no tier 3, three CTAs of 8 warps per SM (24 warps,
// <= 85 registers), for the items that never grow heavy nodes (every seller,
// every put buyer: DESIGN.md section 5); a heavy node there aborts the item,
// which the full kernel re-runs.
#ifndef AMTC_FULL_WARPS
#define AMTC_FULL_WARPS 20
#endif
#ifndef AMTC_FULL_CB
#define AMTC_FULL_CB 3
#endif
constexpr int STRIP_C = AMTC_FULL_CB, STRIP_B = AMTC_FULL_CB, STRIP_WARPS = AMTC_FULL_WARPS, STRIP_MINB = 1;
#ifndef AMTC_LIGHT_CFG
#define AMTC_LIGHT_CFG 6, 6, 8, 3
#endif
constexpr int LIGHT_CFG[4] = {AMTC_LIGHT_CFG};
constexpr int LIGHT_C = LIGHT_CFG[0], LIGHT_B = LIGHT_CFG[1], LIGHT_WARPS = LIGHT_CFG[2], LIGHT_MINB = LIGHT_CFG[3];
// split mode (single trees, small batches): 16 warps with 6-vertex slots --
// a strip pipeline is latency bound, so fewer warps per SM and no arena spills
// of 5-vertex functions beat the 20 / 4 shape there (config 5b: 128 vs 177 ms)
constexpr int SPLIT_C = 6, SPLIT_B = 6, SPLIT_WARPS = 16;
#define SPLIT_KERNEL strip_kernel<SPLIT_C, SPLIT_B, SPLIT_WARPS, 1, true>
#define STRIP_KERNEL strip_kernel<STRIP_C, STRIP_B, STRIP_WARPS, STRIP_MINB, true>
#define LIGHT_KERNEL strip_kernel<LIGHT_C, LIGHT_B, LIGHT_WARPS, LIGHT_MINB, false>
constexpr size_t STRIP_SMEM = sizeof(CtaHdr) + sizeof(StripSmem<STRIP_C, STRIP_B, true>) * STRIP_WARPS;
constexpr size_t LIGHT_SMEM = sizeof(CtaHdr) + sizeof(StripSmem<LIGHT_C, LIGHT_B, false>) * LIGHT_WARPS;
constexpr size_t SPLIT_SMEM = sizeof(CtaHdr) + sizeof(StripSmem<SPLIT_C, SPLIT_B, true>) * SPLIT_WARPS;

static int strip_set_smem() {
    static int done = 0;
    if (!done) {
        if (cudaFuncSetAttribute(STRIP_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)STRIP_SMEM) !=
            cudaSuccess)
            return STATUS_ECUDA;
        if (cudaFuncSetAttribute(LIGHT_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LIGHT_SMEM) !=
            cudaSuccess)
            return STATUS_ECUDA;
        if (cudaFuncSetAttribute(SPLIT_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SPLIT_SMEM) !=
            cudaSuccess)
            return STATUS_ECUDA;
        done = 1;
    }
    return STATUS_OK;
}

static int g_tl_override = 0;  // testing hook (amtc_debug_set_heavy_threshold)
void strip_set_heavy_threshold(int tl) { g_tl_override = tl > 0 ? tl : 0; }
static int g_cap_shift = 0;  // testing hook (amtc_debug_set_arena_shift): arenas >> shift
void strip_set_arena_shift(int sh) { g_cap_shift = sh > 0 ? (sh > 16 ? 16 : sh) : 0; }

StripCaps strip_caps(int N, int level) {
    // level 0: first pass; each retry level quadruples the arenas
    StripCaps c;
    c.C = STRIP_C;
    c.B = STRIP_B;
    c.BG = 256;
    c.TL = g_tl_override ? g_tl_override : 64;
    const int64_t mul = (int64_t)1 << (2 * level);
    auto clampi = [](int64_t v) { return (int)(v > ((int64_t)1 << 28) ? ((int64_t)1 << 28) : v); };
    // arenas sized so that the heaviest config-4 items (call buyers at k/h ~ 15:
    // ~16 heavy columns of up to ~3N vertices) never need a retry pass: the
    // row arena holds one level of a strip, the carry arena every carried
    // function of a strip (the band crosses a carry column for ~32 levels)
    c.rarena_cap = clampi(mul * (64 * (int64_t)(N + 2) + 8192) >> g_cap_shift);
    c.carena_cap = clampi(mul * (100 * (int64_t)(N + 2) + 8192) >> g_cap_shift);
    // tier 3 scratch: stage + W (<= 2 (nU + nD) + 8 vertices; the sawtooth grows by
    // two vertices per level, so nU, nD <= ~2N) + block minima
    c.hscr_cap = clampi(heavy::STAGE * 32 + mul * (14 * (int64_t)(N + 2) + 4096));
    c.zbuf_cap = clampi(mul * (6 * (int64_t)(N + 2) + 4096));
    return c;
}

// the light kernel: no tier 3, small arenas (its functions stay below ~10 vertices)
static StripCaps strip_caps_light(int N) {
    StripCaps c = strip_caps(N, 0);
    c.C = LIGHT_C;
    c.B = LIGHT_B;
    c.rarena_cap = 8 * (N + 2) + 4096;
    c.carena_cap = 8 * (N + 2) + 4096;
    c.hscr_cap = 0;
    c.zbuf_cap = 0;
    return c;
}

void strip_tc_caps(int N, int level, int& rarena, int& carena, int& hscr, int& zbuf, int& tl) {
    const StripCaps c = strip_caps(N, level);
    rarena = c.rarena_cap;
    carena = c.carena_cap;
    hscr = c.hscr_cap;
    zbuf = c.zbuf_cap;
    tl = c.TL;
}

size_t strip_ws_bytes_per_warp(int N, int level) { return strip_layout(N, strip_caps(N, level)).total; }
size_t strip_ws_bytes_per_warp_light(int N) { return strip_layout(N, strip_caps_light(N)).total; }
static StripCaps strip_caps_split(int N) {
    StripCaps c = strip_caps(N, 0);
    c.C = SPLIT_C;
    c.B = SPLIT_B;
    return c;
}
size_t strip_ws_bytes_per_warp_split(int N) { return strip_layout(N, strip_caps_split(N)).total; }
int strip_split_warps_per_cta() { return SPLIT_WARPS; }
int strip_light_warps_per_cta() { return LIGHT_WARPS; }
int strip_light_ctas_per_sm() {
    int b = 0;
    if (strip_set_smem() != STATUS_OK) return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, LIGHT_KERNEL, LIGHT_WARPS * 32, LIGHT_SMEM);
    return b;
}

// split mode: bytes of one strip's carry column (chdr | csl | cv) and the
// per-tree carry arena (vertices)
size_t strip_carry_bytes(int N) {
    return align256(sizeof(int2) * (size_t)(N + 2)) + align256(sizeof(double) * (size_t)(N + 2)) +
           align256(sizeof(Vtx) * (size_t)SPLIT_C * (size_t)(N + 2));
}
int strip_split_arena_cap(int N) {
    const int64_t v = 16 * (int64_t)(N + 2) * (N / SW + 1) + 65536;
    return (int)std::min<int64_t>(v, (int64_t)1 << 30);
}
size_t strip_vtx_bytes() { return sizeof(Vtx); }

int strip_warps_per_cta() { return STRIP_WARPS; }

int strip_ctas_per_sm() {
    int b = 0;
    if (strip_set_smem() != STATUS_OK) return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, STRIP_KERNEL, STRIP_WARPS * 32, STRIP_SMEM);
    return b;
}

int strip_launch(const StripLaunchArgs& a, cudaStream_t s) {
    StripLaunch L;
    L.in = a.in;
    L.N = a.N;
    L.out = a.out;
    L.items = a.items;
    L.n_items = a.n_items;
    L.work_counter = a.work_counter;
    L.ovf_items = a.ovf_items;
    L.ovf_count = a.ovf_count;
    L.vertex_sum = a.vertex_sum;
    L.ws = a.ws;
    L.split_S = a.split_S;
    L.progress = a.progress;
    L.carry = a.carry;
    L.carry_stride = a.carry_stride;
    L.c_csl = align256(sizeof(int2) * (size_t)(a.N + 2));
    L.c_cv = L.c_csl + align256(sizeof(double) * (size_t)(a.N + 2));
    L.carena_split = reinterpret_cast<Vtx*>(a.carena_split);
    L.carena_cnt = a.carena_cnt;
    L.carena_split_cap = a.carena_split_cap;
    L.item_lo = a.item_lo;
    L.peer_strip = a.peer_strip;
    L.sys_fence = a.sys_fence;
    L.peer_carry = a.peer_carry;
    L.peer_carena = reinterpret_cast<Vtx*>(a.peer_carena);
    L.peer_progress = a.peer_progress;
    L.hedge = a.hedge;
    L.caps = a.light ? strip_caps_light(a.N) : (a.split_S > 0 ? strip_caps_split(a.N) : strip_caps(a.N, a.level));
    L.lay = strip_layout(a.N, L.caps);
    if (L.lay.total != a.ws_stride) return STATUS_EINVAL;
    if (strip_set_smem() != STATUS_OK) return STATUS_ECUDA;
    if (a.light) LIGHT_KERNEL<<<a.ctas, LIGHT_WARPS * 32, LIGHT_SMEM, s>>>(L);
    else if (a.split_S > 0) SPLIT_KERNEL<<<a.ctas, SPLIT_WARPS * 32, SPLIT_SMEM, s>>>(L);
    else STRIP_KERNEL<<<a.ctas, STRIP_WARPS * 32, STRIP_SMEM, s>>>(L);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STATUS_OK : STATUS_ECUDA;
}

}  // namespace amtc
