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
//     pass-A result above B) aborts the item, which the full kernel re-runs.
#include <cuda_runtime.h>

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
#define AMTC_L2_WARPS 8
#endif
#ifndef AMTC_L2_MINB
#define AMTC_L2_MINB 2
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

template <int C, int B>
struct LightSmem {
    Vtx row[C * LW];  // vertex i of column c at row[i * LW + c]
    Vtx scr[B * 32];  // pass-1 scratch (A) of lane l: scr[i * 32 + l]
    double csl[2];    // left-tail slopes of carry columns 32, 33
    int cn[2];        // their vertex counts
};

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
};


template <int C, int B, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) light_kernel(const __grid_constant__ LightLaunch L) {
    static_assert(2 + 3 * C <= 32, "one lane per double of a carry record");
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    LightSmem<C, B>& S = reinterpret_cast<LightSmem<C, B>*>(smem_raw)[wib];
    const int N = L.N;
    LCarry<C>* const carry0 =
        reinterpret_cast<LCarry<C>*>(L.ws + (size_t)(blockIdx.x * WARPS + wib) * L.ws_stride);
    // per-lane global scratch for the rare pass-A result wider than B vertices
    Vtx* const gscr = reinterpret_cast<Vtx*>(L.ws + (size_t)(blockIdx.x * WARPS + wib) * L.ws_stride +
                                             light2_carry_bytes<C>(N)) + (size_t)lane * LBG;
    const int item_lo = L.item_lo ? *L.item_lo : 0;
    for (;;) {
        int it = 0;
        if (lane == 0) it = item_lo + atomicAdd(L.work_counter, 1);
        it = __shfl_sync(LFULL, it, 0);
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
        int my_n = 1;
        double my_sl = 0.0;

        for (int s = N / 32; s >= 0; --s) {
            const int j0 = 32 * s, j = j0 + lane;
            LCarry<C>* const cout = carry0 + (size_t)(s & 1) * (N + 2);              // column 32 s, per level
            const LCarry<C>* const cin = carry0 + (size_t)((s + 1) & 1) * (N + 2);   // column 32 (s + 1)
            // a2: leaves t = N+1, payoff (0,0): z = y^- S^a - y^+ S^b, discounted (A11)
            {
                const double dN1 = exp(-oc.rho * (double)(N + 1));
                const double Sd = oc.S0 * exp(oc.h * (double)((N + 1) - 2 * j)) * dN1;
                S.row[lane] = Vtx{0.0, 0.0, -km * Sd};
                my_n = 1;
                my_sl = -kp * Sd;
                if (lane == 31) {  // lane 31's down child at t = N: the leaf (N+1, j+1)
                    const double Sd1 = oc.S0 * exp(oc.h * (double)((N + 1) - 2 * (j + 1))) * dN1;
                    const int par = (N + 1) & 1;
                    S.row[32 + par] = Vtx{0.0, 0.0, -km * Sd1};
                    S.cn[par] = 1;
                    S.csl[par] = -kp * Sd1;
                }
            }
            // node quote S_{t,j} and discount r^-t at t = N, then one multiply per level
            double Sq = oc.S0 * exp(oc.h * (double)(N - 2 * j));
            double disc = exp(-oc.rho * (double)N);
            const bool has_right = s < N / 32;
            double pre = 0.0;  // this lane's double of the next level's carry record
            const int t_end = max(j0, 1);
            for (int t = N; t >= t_end; --t) {
                // carry of level t+1 (loaded during level t+1) -> column 32 + ((t+1) & 1)
                if (t < N && has_right && t + 1 >= j0 + 32) {
                    const int par = (t + 1) & 1;
                    if (lane == 0) S.csl[par] = pre;
                    else if (lane == 1) S.cn[par] = __double2loint(pre);
                    else if (lane < 2 + 3 * C) {
                        const int q = lane - 2;
                        (&S.row[(q / 3) * LW + 32 + par].x)[q % 3] = pre;
                    }
                }
                // prefetch the record of level t (lane 31's down child at level t-1)
                if (has_right && t >= j0 + 32 && lane < 2 + 3 * C) pre = cin[t].d[lane];
                __syncwarp();
                const bool active = j <= t;
                int dn = __shfl_down_sync(LFULL, my_n, 1);
                double dsl = __shfl_down_sync(LFULL, my_sl, 1);
                const int dcol = lane < 31 ? lane + 1 : 32 + ((t + 1) & 1);
                if (lane == 31) {
                    dn = S.cn[(t + 1) & 1];
                    dsl = S.csl[(t + 1) & 1];
                }
                // node constants: quotes (discounted), exercise function u_t (P:96 / P:133)
                const double Sd = Sq * disc;
                const double lo = -kp * Sd, hi = -km * Sd;
                double xi, zeta;
                option_payoff(oc, Sq, xi, zeta);
                const double ux = seller ? zeta : -zeta;
                double uf = (seller ? xi : -xi) * disc;
                if (euro && t < N) uf = seller ? -1e300 : 1e300;  // NEXT #3: no exercise before N
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
                        e = lane_pass2<LW>(A, lo, hi, ux, uf, seller, E);
                    } else {
                        const FnT<1> A = make_fn_s<1>(gscr + (LBG - nA), nA, slA);
                        e = lane_pass2<LW>(A, lo, hi, ux, uf, seller, E);
                    }
                    my_n = E.m;
                    my_sl = E.sl;
                }
                if (active) {
                    err |= e;
                    maxn = max(maxn, my_n);
                    vsum += (unsigned long long)my_n;
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
                }
                Sq *= e_h;
                disc *= e_r;
            }
            err = __reduce_or_sync(LFULL, err);
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
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(LFULL, vsum, o);
        if (lane == 0) {
            atomicAdd(L.vertex_sum, vsum);
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
#define LIGHT2_KERNEL light_kernel<L2_C, L2_B, L2_WARPS, L2_MINB>
constexpr size_t L2_SMEM = sizeof(LightSmem<L2_C, L2_B>) * L2_WARPS;

static int light2_set_smem() {
    static int done = 0;
    if (!done) {
        if (cudaFuncSetAttribute(LIGHT2_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L2_SMEM) !=
            cudaSuccess)
            return STATUS_ECUDA;
        done = 1;
    }
    return STATUS_OK;
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
    if (a.ws_stride != light2_ws_bytes_per_warp(a.N)) return STATUS_EINVAL;
    if (light2_set_smem() != STATUS_OK) return STATUS_ECUDA;
    LIGHT2_KERNEL<<<a.ctas, L2_WARPS * 32, L2_SMEM, s>>>(L);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STATUS_OK : STATUS_ECUDA;
}

}  // namespace amtc
