// amtc_tc2.cu -- SMEM-resident transaction-cost solver (the main TC path).
//
// One CTA per work item (option, party); persistent grid pulling items from
// the heavy-first queue.  The whole tree level lives in shared memory and is
// updated IN PLACE, level by level (t = N .. 1), as the paper's recursion
// requires (Sec. 4.1 tree):
//   * every node j has a descriptor (vertex count, big-arena offset or -1) and
//     an inline slot of KS vertices; functions with more than KS vertices live
//     in a per-CTA global "big" arena (ping-pong per level);
//   * the left-tail slope of every z_{t,j} is the quote slope lo_{t,j}
//     (SURVEY A.3), so it is recomputed, never stored;
//   * phase L: threads take nodes j = tid + k*T and run the sequential node
//     update (pwl_device.cuh) with thread-local scratch; a node whose children
//     hold more than HEAVY_T vertices in total is queued instead;
//   * phase H: each warp takes queued heavy nodes and runs the warp-cooperative
//     update (pwl_warp.cuh), writing into the big arena;
//   * phase W (after a barrier, since node j-1 reads slot j): results land in
//     the slots / descriptors.
// Capacity overflow (arena, scratch) aborts the item; the host re-runs it with
// larger arenas, and finally on the global-memory solver (amtc_tc.cu).
#include <cuda_runtime.h>

#include "amtc_internal.cuh"
#include "pwl_device.cuh"
#include "pwl_warp.cuh"

namespace amtc {

constexpr int TC2_THREADS = 512;
constexpr int TC2_WARPS = TC2_THREADS / 32;
constexpr int HEAVY_T = 24;              // nU + nD above this -> warp-cooperative
constexpr int LSCR = 2 * HEAVY_T + 16;   // thread-local scratch vertices per buffer
constexpr int MAXP = 4;                  // nodes per thread per level -> N + 1 <= 2048

struct OptC {
    double S0, K, K2, k, h, rho;
    int kind;
};

__device__ __forceinline__ int tc2_validate(const BatchPtrs& in, int64_t i, int N, OptC& oc) {
    oc.S0 = in.S0[i];
    oc.K = in.K[i];
    oc.K2 = in.K2 ? in.K2[i] : 0.0;
    const double T = in.T[i], sigma = in.sigma[i], R = in.R[i];
    oc.k = in.k ? in.k[i] : 0.0;
    oc.kind = in.kind[i];
    if (!(oc.S0 > 0.0) || !(T > 0.0) || !(sigma > 0.0) || N < 1) return STATUS_EINVAL;
    if (!(oc.k >= 0.0 && oc.k < 1.0)) return STATUS_EINVAL;
    if (oc.kind != KIND_PUT && oc.kind != KIND_CALL && oc.kind != KIND_BULL) return STATUS_EINVAL;
    if (oc.kind != KIND_BULL && !(oc.K > 0.0)) return STATUS_EINVAL;
    if (oc.kind == KIND_BULL && !(oc.K < oc.K2)) return STATUS_EINVAL;
    if (!isfinite(R)) return STATUS_EINVAL;
    oc.h = sigma * sqrt(T / (double)N);
    oc.rho = R * T / (double)N;
    if (!(oc.rho < oc.h && -oc.h < oc.rho)) return STATUS_EARBITRAGE;
    return STATUS_OK;
}

__device__ __forceinline__ void tc2_payoff(const OptC& oc, double S, double& xi, double& zeta) {
    if (oc.kind == KIND_PUT) { xi = oc.K; zeta = -1.0; }                       // (K, -1)
    else if (oc.kind == KIND_CALL) { xi = -oc.K; zeta = 1.0; }                 // (-K, +1) reading R6
    else { xi = fmax(S - oc.K, 0.0) - fmax(S - oc.K2, 0.0); zeta = 0.0; }
}

size_t tc2_smem_bytes(int N, int KS) {
    const size_t nn = (size_t)N + 2;
    return nn * sizeof(int2) + nn * KS * sizeof(Vtx) + nn * 3 * sizeof(int) + 64;
}

size_t tc2_workspace_bytes(int N, int big_cap, int heavy_scr) {
    size_t tables = sizeof(double) * (size_t)(2 * N + 3 + N + 2);
    tables = (tables + 255) & ~(size_t)255;
    return tables + sizeof(Vtx) * (2 * (size_t)big_cap + (size_t)TC2_WARPS * heavy_scr);
}

template <int KS>
__global__ void __launch_bounds__(TC2_THREADS, 1) tc2_kernel(Tc2Launch L) {
    extern __shared__ __align__(16) char smem[];
    const int N = L.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nn = N + 2;
    int2* desc = reinterpret_cast<int2*>(smem);                          // (count, big offset | -1)
    Vtx* slots = reinterpret_cast<Vtx*>(smem + sizeof(int2) * nn);      // nn * KS
    int* hq = reinterpret_cast<int*>(slots + (size_t)nn * KS);            // heavy queue
    int* hn = hq + nn;                                                    // heavy result counts
    int* ho = hn + nn;                                                    // heavy result offsets
    __shared__ int s_item, s_err, s_maxn, s_hcount, s_big[2];

    char* base = L.ws + (size_t)blockIdx.x * L.ws_stride;
    double* Epow = reinterpret_cast<double*>(base);
    double* Dpow = Epow + (2 * N + 3);
    size_t tables = sizeof(double) * (size_t)(2 * N + 3 + N + 2);
    tables = (tables + 255) & ~(size_t)255;
    Vtx* big[2] = {reinterpret_cast<Vtx*>(base + tables), reinterpret_cast<Vtx*>(base + tables) + L.big_cap};
    Vtx* hscr = big[1] + L.big_cap + (size_t)warp * L.heavy_scr;

    Vtx r0[LSCR], r1[LSCR];        // thread-local scratch of the sequential update
    Vtx hold[MAXP][KS];            // light results waiting for phase W
    int hold_n[MAXP], hold_off[MAXP];

    for (;;) {
        if (tid == 0) {
            s_item = atomicAdd(L.work_counter, 1);
            s_err = 0;
            s_maxn = 1;
        }
        __syncthreads();
        const int it = s_item;
        if (it >= *L.n_items) break;
        const int code = L.items[it];
        const int64_t opt = code >> 1;
        const int party = code & 1;
        OptC oc;
        if (tc2_validate(L.in, opt, N, oc) != STATUS_OK) {
            __syncthreads();
            continue;
        }
        for (int i = tid; i < 2 * N + 3; i += TC2_THREADS) Epow[i] = exp(oc.h * (double)(i - (N + 1)));
        for (int t = tid; t < N + 2; t += TC2_THREADS) Dpow[t] = exp(-oc.rho * (double)t);
        if (tid == 0) { s_big[0] = 0; s_big[1] = 0; s_hcount = 0; }
        __syncthreads();
        const double kp = 1.0 + oc.k, km = 1.0 - oc.k;
        // a2: leaves t = N+1, payoff (0,0)  (Alg. 1 line 5)
        for (int j = tid; j <= N + 1; j += TC2_THREADS) {
            const double Sd = oc.S0 * Epow[(N + 1) - 2 * j + (N + 1)] * Dpow[N + 1];
            desc[j] = make_int2(1, -1);
            Vtx& v = slots[(size_t)j * KS];
            v.x = 0.0;
            v.f = 0.0;
            v.s = -km * Sd;
        }
        __syncthreads();
        int cur = 0;  // big arena holding level t+1
        unsigned long long my_vertices = 0;
        for (int t = N; t >= 1; --t) {
            const double disc = Dpow[t];
            const double discc = Dpow[t + 1];
            const int nxt = cur ^ 1;
            // ---- phase L ----
            int np = 0;
            int lerr = DEV_OK;
            for (int j = tid; j <= t; j += TC2_THREADS, ++np) {
                hold_n[np] = -1;  // -1 = heavy (queued)
                const int2 dU = desc[j], dD = desc[j + 1];
                if (dU.x + dD.x > HEAVY_T) {
                    hq[atomicAdd(&s_hcount, 1)] = j;
                    continue;
                }
                const double SU = oc.S0 * Epow[(t + 1) - 2 * j + (N + 1)];
                const double SD = oc.S0 * Epow[(t + 1) - 2 * (j + 1) + (N + 1)];
                Fn U{dU.y < 0 ? &slots[(size_t)j * KS] : big[cur] + dU.y, dU.x, -kp * SU * discc};
                Fn D{dD.y < 0 ? &slots[(size_t)(j + 1) * KS] : big[cur] + dD.y, dD.x, -kp * SD * discc};
                const double S = oc.S0 * Epow[t - 2 * j + (N + 1)];
                const double lo = -kp * S * disc, hi = -km * S * disc;
                double xi, zeta;
                tc2_payoff(oc, S, xi, zeta);
                int nZ;
                double slZ;
                int e = node_update(U, D, lo, hi, party == 0 ? zeta : -zeta, (party == 0 ? xi : -xi) * disc,
                                    party == 0, r0, r1, LSCR, nZ, slZ);
                if (e == DEV_OVERFLOW) {  // scratch too small: hand it to a warp
                    hq[atomicAdd(&s_hcount, 1)] = j;
                    continue;
                }
                lerr |= e;
                hold_n[np] = nZ;
                my_vertices += (unsigned long long)nZ;
                if (nZ <= KS) {
                    hold_off[np] = -1;
                    for (int q = 0; q < KS; ++q)
                        if (q < nZ) hold[np][q] = r1[q];
                } else {
                    const int off = atomicAdd(&s_big[nxt], nZ);
                    if (off + nZ > L.big_cap) {
                        lerr |= DEV_OVERFLOW;
                    } else {
                        for (int q = 0; q < nZ; ++q) big[nxt][off + q] = r1[q];
                        hold_off[np] = off;
                    }
                    atomicMax(&s_maxn, nZ);
                }
            }
            if (lerr) atomicOr(&s_err, lerr);
            __syncthreads();
            // ---- phase H ----
            const int nh = s_hcount;
            for (int q = warp; q < nh; q += TC2_WARPS) {
                const int j = hq[q];
                const int2 dU = desc[j], dD = desc[j + 1];
                const double SU = oc.S0 * Epow[(t + 1) - 2 * j + (N + 1)];
                const double SD = oc.S0 * Epow[(t + 1) - 2 * (j + 1) + (N + 1)];
                Fn U{dU.y < 0 ? &slots[(size_t)j * KS] : big[cur] + dU.y, dU.x, -kp * SU * discc};
                Fn D{dD.y < 0 ? &slots[(size_t)(j + 1) * KS] : big[cur] + dD.y, dD.x, -kp * SD * discc};
                const double S = oc.S0 * Epow[t - 2 * j + (N + 1)];
                const double lo = -kp * S * disc, hi = -km * S * disc;
                double xi, zeta;
                tc2_payoff(oc, S, xi, zeta);
                int off = 0, nZ = 0;
                int e;
                if (22 * (U.n + D.n) + 2300 > L.heavy_scr) {
                    e = DEV_OVERFLOW;
                } else {
                    e = warp_node_update(U, D, lo, hi, party == 0 ? zeta : -zeta, (party == 0 ? xi : -xi) * disc,
                                         party == 0, hscr, L.heavy_scr, big[nxt], &s_big[nxt], L.big_cap, off, nZ,
                                         lane);
                }
                if (lane == 0) {
                    if (e) atomicOr(&s_err, e);
                    hn[q] = nZ;
                    ho[q] = off;
                    my_vertices += (unsigned long long)nZ;
                    atomicMax(&s_maxn, nZ);
                }
            }
            __syncthreads();
            if (s_err) break;
            // ---- phase W ----
            np = 0;
            for (int j = tid; j <= t; j += TC2_THREADS, ++np) {
                const int n = hold_n[np];
                if (n < 0) continue;
                if (n <= KS) {
                    desc[j] = make_int2(n, -1);
                    for (int q = 0; q < KS; ++q)
                        if (q < n) slots[(size_t)j * KS + q] = hold[np][q];
                } else {
                    desc[j] = make_int2(n, hold_off[np]);
                }
            }
            for (int q = tid; q < nh; q += TC2_THREADS) desc[hq[q]] = make_int2(hn[q], ho[q]);
            if (tid == 0) {
                s_hcount = 0;
                s_big[cur] = 0;  // level t+1's arena is dead after this level
            }
            __syncthreads();
            cur = nxt;
        }
        // a6: root, t = 0, no costs: v_0(y) = min_b [w_0(b) + S0 b] - S0 y
        if (!s_err && warp == 0) {
            const double S1U = oc.S0 * Epow[1 + (N + 1)], S1D = oc.S0 * Epow[-1 + (N + 1)];
            const int2 dU = desc[0], dD = desc[1];
            Fn U{dU.y < 0 ? &slots[0] : big[cur] + dU.y, dU.x, -kp * S1U * Dpow[1]};
            Fn D{dD.y < 0 ? &slots[KS] : big[cur] + dD.y, dD.x, -kp * S1D * Dpow[1]};
            // W into the heavy scratch of warp 0, merged cooperatively
            int nW = 0;
            double slW = 0.0;
            const int nE = U.n + D.n;
            int e = (6 * nE + 200 > L.heavy_scr) ? DEV_OVERFLOW
                                                 : warp_merge_max(U, D, hscr, hscr + 2 * nE + 64, 2 * nE + 2, nW,
                                                                  slW, lane);
            double mv = INFINITY;
            if (!e) {
                const Vtx* Wv = hscr + 2 * nE + 64;
                for (int i = lane; i < nW; i += 32) mv = fmin(mv, fma(oc.S0, Wv[i].x, Wv[i].f));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mv = fmin(mv, __shfl_xor_sync(FULL, mv, o));
                if (!(slW + oc.S0 < 0.0) || !(Wv[nW - 1].s + oc.S0 > 0.0)) e = DEV_UNBOUNDED;
            }
            if (lane == 0) {
                double xi, zeta;
                tc2_payoff(oc, oc.S0, xi, zeta);
                const double intrinsic = xi + zeta * oc.S0;
                if (e) s_err |= e;
                else if (party == 0) L.out[opt].ask = fmax(intrinsic, mv);
                else L.out[opt].bid = fmax(intrinsic, -mv);
            }
        }
        if (my_vertices) atomicAdd(L.vertex_sum, my_vertices);
        __syncthreads();
        if (tid == 0) {
            if (s_err & DEV_OVERFLOW) {
                const int k = atomicAdd(L.ovf_count, 1);
                L.ovf_items[k] = code;
            } else if (s_err & DEV_UNBOUNDED) {
                atomicMax(&L.out[opt].status, STATUS_EUNBOUNDED);
            }
            atomicMax(&L.out[opt].max_bp, s_maxn);
        }
        __syncthreads();
    }
}

int tc2_max_n() { return TC2_THREADS * MAXP - 1; }

// KS for a given N so that the level fits 227 KB of shared memory
int tc2_pick_ks(int N) {
    const size_t lim = 227 * 1024;
    for (int ks = 4; ks >= 1; --ks)
        if (tc2_smem_bytes(N, ks) <= lim) return ks;
    return 0;
}

int tc2_launch(const Tc2Launch& L, int grid, cudaStream_t s) {
    const int ks = tc2_pick_ks(L.N);
    if (ks == 0 || L.N > tc2_max_n()) return STATUS_EINVAL;
    const size_t sm = tc2_smem_bytes(L.N, ks);
    cudaError_t e = cudaSuccess;
    switch (ks) {
#define CASE(K)                                                                                   \
    case K:                                                                                       \
        e = cudaFuncSetAttribute(tc2_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        if (e != cudaSuccess) return STATUS_ECUDA;                                                \
        tc2_kernel<K><<<grid, TC2_THREADS, sm, s>>>(L);                                           \
        break;
        CASE(1) CASE(2) CASE(3) CASE(4)
#undef CASE
    }
    note_launch();
    return STATUS_OK;
}

}  // namespace amtc
