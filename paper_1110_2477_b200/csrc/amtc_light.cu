// amtc_light.cu -- the LIGHT transaction-cost solver: one warp per work item
// (option, party) whose node functions stay small (the seller of a put or a
// call, the buyer of a put: DESIGN.md section 5), swept in 32-column strips
// right to left exactly as the full solver (amtc_strip.cu; Sec. 3,
// P:94-144, on the tree of Sec. 4.1; region-B dependency P:164-166).
//
// What differs from the full kernel's strip loop (same node algebra,
// pwl_lane.cuh, instantiated with compile-time strides):
//   * every function of the strip lives in ONE shared-memory matrix
//     row[i * LW + c] (vertex i of column c): columns 0..31 are the lanes'
//     functions, columns 32 / 33 (by level parity) hold lane 31's down child
//     -- the carry column of the strip to the right -- so every lane reads its
//     children (column lane, column lane+1) with the same shared-memory code;
//   * the carry column is prefetched one level ahead (each lane loads one
//     double of the next level's record, stores it a level later), so no level
//     waits on a global load;
//   * node quotes S_{t,j} r^-t are carried by one multiply per level (no
//     per-option tables);
//   * no arenas and no tiers: a function with more than C vertices (or a
//     pass-A result above B) aborts the item, which the full kernel re-runs;
//   * split mode (SPLIT = true; single trees and small batches of light
//     trees, e.g. config 5b): every strip of a tree is its own work item, the
//     strips run on different warps and are pipelined through a per-(tree,
//     strip) carry column in HBM and a progress counter (the level the strip
//     has published); the consumer waits for level t while it is still
//     computing level t+1 (the record is staged one level ahead), so the
//     hand-off overlaps the node updates.
#include <cuda_runtime.h>

#include <climits>

#include "amtc_internal.cuh"
#include "amtc_option.cuh"
#include "pwl_device.cuh"
#include "pwl_heavy.cuh"
#include "pwl_lane.cuh"
#include "amtc_root.cuh"

namespace amtc {

// shape (developer sweeps: -DAMTC_L2_WARPS=8 etc.): C-vertex function slots,
// B-vertex pass-A scratch, WARPS per CTA, MINB CTAs per SM; GFALLBACK: a pass-A
// result above B vertices goes to a per-lane global scratch instead of
// aborting the item.  Measured on config-4 puts (1184 options, N=1500; the
// strip kernel's light variant: 338 ms): B=10 / 8 warps x 2 / no fallback
// 160 ms, B=8 with fallback 267 ms, B=6 / 12 warps 319 ms, B=8 without
// fallback 567 ms (211 items overflow into a re-run pass).
#ifndef AMTC_L2_C
#define AMTC_L2_C 6
#endif
#ifndef AMTC_L2_GFALLBACK
#define AMTC_L2_GFALLBACK 0
#endif
#ifndef AMTC_L2_B
#define AMTC_L2_B 10
#endif
#ifndef AMTC_L2_WARPS
#define AMTC_L2_WARPS 6  // 12 warps / SM at 168 registers: whole config-4 batch 9.24 -> 9.02 s (8 warps, 128 regs)
#endif
#ifndef AMTC_L2_MINB
#define AMTC_L2_MINB 2
#endif
// split mode: a strip publishes its progress every AMTC_L2_PUB levels (one
// __threadfence per publication)
#ifndef AMTC_L2_PUB
#define AMTC_L2_PUB 4
#endif
constexpr int LW = 34;  // columns of the strip matrix: 32 lanes + 2 carry columns
constexpr unsigned LFULL = 0xffffffffu;

// one level of a strip's carry column in global memory, as doubles:
// [0] left-tail slope, [1] vertex count (int bits), [2 + 3 i + c] vertex i (x, f, s)
template <int C>
struct LCarry {
    double d[2 + 3 * C];
};

constexpr int LBG = 64;  // vertices of a lane's global pass-A scratch

template <int C>
__host__ __device__ inline size_t light2_carry_bytes(int N) {
    return (2 * sizeof(LCarry<C>) * (size_t)(N + 2) + 255) & ~(size_t)255;
}

// per-item constants of the warp's current item, kept in shared memory and
// read with volatile loads inside the level loop: in registers they were
// spilled to local memory and reloaded from L2 at every level (the L1 left
// beside 200 KB of shared memory is too small for 16 warps' stacks)
struct LightItem {
    double kp, km, e_h, e_r, S0, K, K2;
    int kind;
    unsigned flags;
    int seller, euro;
};

template <int C, int B>
struct LightSmem {
    Vtx row[C * LW];  // vertex i of column c at row[i * LW + c]
    Vtx scr[B * 32];  // pass-1 scratch (A) of lane l: scr[i * 32 + l]
    double csl[2];    // left-tail slopes of carry columns 32, 33
    double cnd[2];    // their vertex counts (low 32 bits)
    __align__(16) double stg[2][2 + 3 * C];  // carry records staged by cp.async (by level parity)
    LightItem it;
};

template <class T>
__device__ __forceinline__ T vld(const T& x) { return *(const volatile T*)&x; }

// developer instrumentation (-DAMTC_L2_PROF=1, split mode): per-warp clock64
// accumulators summed into g_lprof, read through amtc_debug_full_profile:
// [0] cycles in the level loop, [1] cycles in blocking waits for the strip to
// the right, [2] blocking waits, [3] levels, [4] records staged early
#ifndef AMTC_L2_PROF
#define AMTC_L2_PROF 0
#endif
__device__ unsigned long long g_lprof[8];

// one double global -> shared without a register (cp.async, L1-bypassing 8-byte copy)
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
// 16 bytes global -> shared through L2 only (.cg): the record may have been
// written by another SM after this SM's L1 cached a neighbouring record
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// bytes of one carry column in split mode (N + 2 records)
template <int C>
__host__ __device__ inline size_t light2_col_bytes(int N) {
    return (sizeof(LCarry<C>) * (size_t)(N + 2) + 255) & ~(size_t)255;
}

struct LightLaunch {
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
    size_t ws_stride;
    double* hedge;
    // split mode: strips per tree, per-(tree, strip) progress counters and carry columns
    int split_S;
    int* progress;
    char* carry;
    size_t carry_stride;
};


template <int C, int B, int WARPS, int MINB, bool SPLIT>
__global__ void __launch_bounds__(WARPS * 32, MINB) light_kernel(const __grid_constant__ LightLaunch L) {
    static_assert(2 + 3 * C <= 32, "one lane per double of a carry record");
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    LightSmem<C, B>& S = reinterpret_cast<LightSmem<C, B>*>(smem_raw)[wib];
    LightItem& I = S.it;
    const int N = L.N;
    LCarry<C>* const carry0 =
        reinterpret_cast<LCarry<C>*>(L.ws + (size_t)(blockIdx.x * WARPS + wib) * L.ws_stride);
    // per-lane global scratch for the rare pass-A result wider than B vertices
    Vtx* const gscr = reinterpret_cast<Vtx*>(L.ws + (size_t)(blockIdx.x * WARPS + wib) * L.ws_stride +
                                             light2_carry_bytes<C>(N)) + (size_t)lane * LBG;
    const int item_lo = L.item_lo ? *L.item_lo : 0;
    int split_next = wib * (int)gridDim.x + (int)blockIdx.x;  // split mode: next item of this warp
    for (;;) {
        int it = 0;
        if (SPLIT) {
            // strips of a pipeline are latency bound: deal them round-robin over the
            // CTAs (warp w of CTA b takes items w G + b, w G + b + G W, ...) so they
            // spread over every SM instead of filling the first CTAs to launch; each
            // warp takes its items in increasing order, so the lowest unfinished strip
            // always has its producer (a lower item) done or running: no deadlock
            it = item_lo + split_next;
            split_next += gridDim.x * WARPS;
        } else {
            if (lane == 0) it = item_lo + atomicAdd(L.work_counter, 1);
            it = __shfl_sync(LFULL, it, 0);
        }
        if (it >= *L.n_items) break;
        const int code = L.items[it];
        // split mode: item = tree S + strip (one strip); else item = tree (every strip, right to left)
        const int tree = SPLIT ? code / L.split_S : code;  // 2 option + party
        const int s_first = SPLIT ? code % L.split_S : N / 32, s_last = SPLIT ? s_first : 0;
        const int64_t opt = tree >> 1;
        const bool seller = (tree & 1) == 0;
        OptionConsts oc;
        if (validate_option(L.in, opt, N, true, oc) != STATUS_OK) continue;  // status set by prepare
        if (lane == 0) {
            I.kp = 1.0 + oc.k;  // ask / bid factors
            I.km = 1.0 - oc.k;
            I.e_h = exp(-oc.h);
            I.e_r = exp(oc.rho);
            I.S0 = oc.S0;
            I.K = oc.K;
            I.K2 = oc.K2;
            I.kind = oc.kind;
            I.flags = oc.flags;
            I.seller = seller ? 1 : 0;
            I.euro = (oc.flags & FLAG_EUROPEAN) != 0;
        }
        __syncwarp();
        unsigned err = DEV_OK;
        int maxn = 1;
        unsigned vsum = 0;  // < 2^32: at most C vertices per node, N + 1 levels, N / 32 + 1 strips per lane
        int my_n = 1;
        double my_sl = 0.0;

        for (int s = s_first; s >= s_last; --s) {
            const int j0 = 32 * s, j = j0 + lane;
            // column 32 s (written, per level) and column 32 (s + 1) (read): per-warp
            // ping-pong buffers, or the tree's per-strip columns in split mode
            LCarry<C>* const cout =
                SPLIT ? reinterpret_cast<LCarry<C>*>(L.carry + ((size_t)tree * L.split_S + s) * L.carry_stride)
                      : carry0 + (size_t)(s & 1) * (N + 2);
            const LCarry<C>* const cin =
                SPLIT ? reinterpret_cast<const LCarry<C>*>(L.carry + ((size_t)tree * L.split_S + s + 1) * L.carry_stride)
                      : carry0 + (size_t)((s + 1) & 1) * (N + 2);
            const volatile int* const prog_in = SPLIT ? L.progress + (size_t)tree * L.split_S + s + 1 : nullptr;
            volatile int* const prog_out = SPLIT ? L.progress + (size_t)tree * L.split_S + s : nullptr;
            // a2: leaves t = N+1, payoff (0,0): z = y^- S^a - y^+ S^b, discounted (A11)
            {
                const double dN1 = exp(-oc.rho * (double)(N + 1));
                const double Sd = oc.S0 * exp(oc.h * (double)((N + 1) - 2 * j)) * dN1;
                S.row[lane] = Vtx{0.0, 0.0, -vld(I.km) * Sd};
                my_n = 1;
                my_sl = -vld(I.kp) * Sd;
                if (lane == 31) {  // lane 31's down child at t = N: the leaf (N+1, j+1)
                    const double Sd1 = oc.S0 * exp(oc.h * (double)((N + 1) - 2 * (j + 1))) * dN1;
                    const int par = (N + 1) & 1;
                    S.row[32 + par] = Vtx{0.0, 0.0, -vld(I.km) * Sd1};
                    S.cnd[par] = __hiloint2double(0, 1);
                    S.csl[par] = -vld(I.kp) * Sd1;
                }
            }
            // node quote S_{t,j} and discount r^-t at t = N, then one multiply per level
            double Sq = oc.S0 * exp(oc.h * (double)(N - 2 * j));
            double disc = exp(-oc.rho * (double)N);
            const bool has_right = s < N / 32;
            const int t_end = max(j0, 1);
#if AMTC_L2_PROF
            long long pw = 0, nw = 0, ne = 0;
            const long long p0 = clock64();
#endif
            int seen = INT_MAX;  // split mode: lowest level of strip s+1 known to be published
            bool staged_next = false;  // the record of the next level's down child is already in flight
            for (int t = N; t >= t_end; --t) {
                // the carry record of level t+1 (lane 31's down child now), staged by a
                // cp.async, goes into column 32 + ((t+1) & 1).  Whole-tree mode staged it
                // during level t+1; split mode did so only if strip s+1 had published it
                // by then, else it waits for it here (the record is needed now)
                if (SPLIT && !staged_next && t < N && has_right && t + 1 >= j0 + 32) {
#if AMTC_L2_PROF
                    const long long w0 = clock64();
#endif
                    if (seen > t + 1) {
                        int pv = 0;
                        if (lane == 0) {
                            int spins = 0;  // the producer is usually a level away: spin, then back off
                            while ((pv = *prog_in) > t + 1) {
                                if (++spins > 32) __nanosleep(64);
                            }
                        }
                        seen = __shfl_sync(LFULL, pv, 0);
                        if (seen < 0) {  // strip s+1 failed: finish, the tree is re-run
                            err |= DEV_OVERFLOW;
                            seen = INT_MIN;
                        }
                        __threadfence();
                    }
                    if (lane < (2 + 3 * C) / 2)
                        cp_async16(&S.stg[(t + 1) & 1][2 * lane], &cin[t + 1].d[2 * lane]);
#if AMTC_L2_PROF
                    pw += clock64() - w0;
                    nw += 1;
#endif
                }
                cp_async_wait_all();
                __syncwarp();
                if (t < N && has_right && t + 1 >= j0 + 32 && lane < 2 + 3 * C) {
                    const int par = (t + 1) & 1;
                    const double v = S.stg[par][lane];
                    if (lane == 0) S.csl[par] = v;
                    else if (lane == 1) S.cnd[par] = v;
                    else {
                        const int q = lane - 2;
                        (&S.row[(q / 3) * LW + 32 + par].x)[q % 3] = v;
                    }
                }
                // stage the record of level t (lane 31's down child at level t-1) while
                // level t is computed; split mode only if strip s+1 has published it
                // already (one non-blocking look at its progress), so the node updates
                // of level t never wait for the strip to the right
                staged_next = false;
                if (has_right && t >= j0 + 32) {
                    bool ready = true;
                    if (SPLIT && seen > t) {
                        int pv = 0;
                        if (lane == 0) pv = *prog_in;
                        pv = __shfl_sync(LFULL, pv, 0);
                        if (pv < seen) {
                            seen = pv < 0 ? INT_MIN : pv;
                            if (pv < 0) err |= DEV_OVERFLOW;
                            __threadfence();
                        }
                        ready = seen <= t;
                    }
                    if (ready) {
                        if (lane < (2 + 3 * C) / 2) cp_async16(&S.stg[t & 1][2 * lane], &cin[t].d[2 * lane]);
                        staged_next = true;
#if AMTC_L2_PROF
                        ne += SPLIT ? 1 : 0;
#endif
                    }
                }
                __syncwarp();
                const bool active = j <= t;
                int dn = __shfl_down_sync(LFULL, my_n, 1);
                double dsl = __shfl_down_sync(LFULL, my_sl, 1);
                const int dcol = lane < 31 ? lane + 1 : 32 + ((t + 1) & 1);
                if (lane == 31) {
                    dn = __double2loint(S.cnd[(t + 1) & 1]);
                    dsl = S.csl[(t + 1) & 1];
                }
                // node constants: quotes (discounted), exercise function u_t (P:96 / P:133)
                const double Sd = Sq * disc;
                const double lo = -vld(I.kp) * Sd, hi = -vld(I.km) * Sd;
                const bool sel = vld(I.seller) != 0;
                double ux, uf;
                {
                    OptionConsts pc;  // the payoff's inputs, from shared memory
                    pc.K = vld(I.K);
                    pc.K2 = vld(I.K2);
                    pc.kind = vld(I.kind);
                    pc.flags = vld(I.flags);
                    double xi, zeta;
                    option_payoff(pc, Sq, xi, zeta);
                    ux = sel ? zeta : -zeta;
                    uf = (sel ? xi : -xi) * disc;
                }
                if (vld(I.euro) && t < N) uf = sel ? -1e300 : 1e300;  // NEXT #3: no exercise before N
                int e = DEV_OK, nA = 0;
                double slA = lo;
                bool gA = false;  // A outgrew the shared scratch: it sits in the lane's global scratch
                if (active) {
                    const FnT<LW> U = make_fn_s<LW>(&S.row[lane], my_n, my_sl);
                    const FnT<LW> D = make_fn_s<LW>(&S.row[dcol], dn, dsl);
                    e = lane_pass1<32>(U, D, lo, &S.scr[lane], B, 32, nA, slA);
                    if (AMTC_L2_GFALLBACK && e == DEV_OVERFLOW) {  // rare: W wider than B vertices
                        e = lane_pass1<1>(U, D, lo, gscr, LBG, 1, nA, slA);
                        gA = true;
                    }
                }
                __syncwarp();  // every lane has read its children: the row may be overwritten
                if (active && e == DEV_OK) {
                    EmitT<LW> E;
                    E.out = &S.row[lane];
                    E.cap = C;
                    E.stride = LW;
                    if (!gA) {
                        const FnT<32> A = make_fn_s<32>(&S.scr[lane] + (B - nA) * 32, nA, slA);
                        e = lane_pass2<LW>(A, lo, hi, ux, uf, sel, E);
                    } else {
                        const FnT<1> A = make_fn_s<1>(gscr + (LBG - nA), nA, slA);
                        e = lane_pass2<LW>(A, lo, hi, ux, uf, sel, E);
                    }
                    my_n = E.m;
                    my_sl = E.sl;
                }
                if (active) {
                    err |= (unsigned)e;
                    maxn = max(maxn, my_n);
                    vsum += (unsigned)my_n;
                }
                __syncwarp();
                // carry out: node (t, j0), read by strip s-1's lane 31 at level t-1
                if (s > 0) {
                    const int c_n = __shfl_sync(LFULL, my_n, 0);
                    const double c_sl = __shfl_sync(LFULL, my_sl, 0);
                    double* const rec = cout[t].d;
                    if (lane == 0) rec[0] = c_sl;
                    else if (lane == 1) rec[1] = __hiloint2double(0, c_n);
                    else if (lane < 2 + 3 * min(c_n, C)) {
                        const int q = lane - 2;
                        rec[lane] = (&S.row[(q / 3) * LW].x)[q % 3];
                    }
                    if (SPLIT && (t % AMTC_L2_PUB == 0 || t == t_end)) {  // publish levels >= t to strip s-1
                        __threadfence();
                        __syncwarp();
                        if (lane == 0) *prog_out = t;
                    }
                }
                Sq *= vld(I.e_h);
                disc *= vld(I.e_r);
            }
            cp_async_wait_all();
#if AMTC_L2_PROF
            if (SPLIT && lane == 0) {
                atomicAdd(&g_lprof[0], (unsigned long long)(clock64() - p0));
                atomicAdd(&g_lprof[1], (unsigned long long)pw);
                atomicAdd(&g_lprof[2], (unsigned long long)nw);
                atomicAdd(&g_lprof[3], (unsigned long long)(N - t_end + 1));
                atomicAdd(&g_lprof[4], (unsigned long long)ne);
            }
#endif
            err = __reduce_or_sync(LFULL, err);
            if (SPLIT && err && s > 0 && lane == 0) {  // never leave strip s-1 waiting
                __threadfence();
                *prog_out = -1;
            }
            if (err) break;
            if (s == 0) {
                const Fn mine = make_fn(&S.row[lane], my_n, my_sl, LW);
                err |= tc_root(mine, oc, seller, &L.out[opt],
                               L.hedge ? &L.hedge[2 * opt + (seller ? 0 : 1)] : nullptr, lane);
            }
            __syncwarp();
        }
        // per-item bookkeeping
        err = __reduce_or_sync(LFULL, err);
        maxn = __reduce_max_sync(LFULL, maxn);
        const unsigned long long vtot = __reduce_add_sync(LFULL, vsum);  // < 2^32 per item as well
        if (lane == 0) {
            atomicAdd(L.vertex_sum, vtot);
            if (err & DEV_OVERFLOW) {  // re-run by the full kernel (arenas, tiers)
                const int q = atomicAdd(L.ovf_count, 1);
                L.ovf_items[q] = code;
            } else if (err & DEV_UNBOUNDED) {
                atomicMax(&L.out[opt].status, STATUS_EUNBOUNDED);
            } else {
                atomicMax(&L.out[opt].max_bp, maxn);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
constexpr int L2_C = AMTC_L2_C, L2_B = AMTC_L2_B, L2_WARPS = AMTC_L2_WARPS, L2_MINB = AMTC_L2_MINB;
#define LIGHT2_KERNEL light_kernel<L2_C, L2_B, L2_WARPS, L2_MINB, false>
#define LIGHT2_SPLIT_KERNEL light_kernel<L2_C, L2_B, L2_WARPS, L2_MINB, true>
constexpr size_t L2_SMEM = sizeof(LightSmem<L2_C, L2_B>) * L2_WARPS;

static int light2_set_smem() {
    static int done = 0;
    if (!done) {
        if (cudaFuncSetAttribute(LIGHT2_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L2_SMEM) !=
                cudaSuccess ||
            cudaFuncSetAttribute(LIGHT2_SPLIT_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L2_SMEM) !=
                cudaSuccess)
            return STATUS_ECUDA;
        done = 1;
    }
    return STATUS_OK;
}
size_t light2_split_carry_bytes(int N) { return light2_col_bytes<L2_C>(N); }
int light_profile(unsigned long long out[8], int reset) {
    if (cudaMemcpyFromSymbol(out, g_lprof, sizeof(unsigned long long) * 8) != cudaSuccess) return STATUS_ECUDA;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (cudaMemcpyToSymbol(g_lprof, z, sizeof(z)) != cudaSuccess) return STATUS_ECUDA;
    }
    return AMTC_L2_PROF ? STATUS_OK : STATUS_EINVAL;
}

size_t light2_ws_bytes_per_warp(int N) { return light2_carry_bytes<L2_C>(N) + sizeof(Vtx) * 32 * LBG; }
int light2_warps_per_cta() { return L2_WARPS; }
int light2_ctas_per_sm() {
    int b = 0;
    if (light2_set_smem() != STATUS_OK) return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, LIGHT2_KERNEL, L2_WARPS * 32, L2_SMEM);
    return b;
}

int light2_launch(const StripLaunchArgs& a, cudaStream_t s) {
    LightLaunch L;
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
    L.ws_stride = a.ws_stride;
    L.hedge = a.hedge;
    L.split_S = a.split_S;
    L.progress = a.progress;
    L.carry = a.carry;
    L.carry_stride = a.carry_stride;
    if (a.ws_stride != light2_ws_bytes_per_warp(a.N)) return STATUS_EINVAL;
    if (a.split_S > 0 && a.carry_stride != light2_col_bytes<L2_C>(a.N)) return STATUS_EINVAL;
    if (light2_set_smem() != STATUS_OK) return STATUS_ECUDA;
    if (a.split_S > 0) LIGHT2_SPLIT_KERNEL<<<a.ctas, L2_WARPS * 32, L2_SMEM, s>>>(L);
    else LIGHT2_KERNEL<<<a.ctas, L2_WARPS * 32, L2_SMEM, s>>>(L);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STATUS_OK : STATUS_ECUDA;
}

}  // namespace amtc
