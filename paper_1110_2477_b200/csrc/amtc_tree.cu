// amtc_tree.cu -- ONE large frictionless (k = 0) CRR tree (config 5a: N up to
// 10^5 and beyond), on one GPU or sharded over the GPUs of an NCCL
// communicator.
//
// Recursion (Appendix; no extra level in frictionless mode):
//   V_N(j) = max(P(S_{N,j}), 0),  V_t(j) = max(P(S_{t,j}), p_u V_{t+1}(j) + p_d V_{t+1}(j+1)).
// Node (t, j) needs (t+1, j) and (t+1, j+1): the dependency cone of a band of
// D levels over output columns [j0, j0 + W) is the input window [j0, j0 + W + D)
// at the band's top level (the paper's region-B dependency).
//
// Band kernel: each warp owns M = 16 (or 24) consecutive columns per lane (32 M
// columns, the level in registers); it reads its window at level t_top, runs
// D = 256 levels with one 64-bit shuffle per level (the j+1 neighbour of a
// lane's last column), and writes the first 32 M - D columns of level t_top - D
// (the right D columns become invalid one per level: the ghost zone).  A
// band is one launch; the level lives in HBM/L2 between bands (800 KB at
// N = 10^5).  No shared memory, no __syncthreads: warps are independent.
//
// The exercise value is carried incrementally per column (S_{t,j} = d S_{t+1,j}):
// put X = K - S: X_t = d X_{t+1} + K (1 - d); call X = S - K: X_t = d X_{t+1} - K (1 - d).
// max(X, c) with c = p_u V + p_d V' >= +0 is a signed 64-bit integer max of the
// bit patterns (IEEE order of non-negative doubles = integer order; a negative X
// has a negative pattern), which runs on the integer ALU instead of the FP64
// pipe's slow DMNMX (4.0e12/s vs 1.8e13/s DFMA on B200, profiles/r01_fp64_peak.json).
//
// Sharding (amtc_price_tree_sharded): rank g owns columns
// [ceil(g w / n_a), ceil((g+1) w / n_a)) of the current level (w = t + 1 columns,
// n_a = clamp(w / 4096, 1, n) active ranks: processor reduction, P:286-288;
// re-split every band -- the paper's per-round rebalancing).  Before a
// band each rank gathers its input window from the owners (ncclSend/ncclRecv
// in one group: its own range plus a halo of D columns from the right and the
// re-split shift from the left), then runs the band kernel locally.
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <mutex>
#include <string>

#include <algorithm>
#include <cmath>
#include <vector>

#include "amtc.h"
#include "amtc_internal.cuh"

namespace amtc {

// band shapes (measured on B200): 16 columns per lane and 256 levels per band
// for N <= 3e5 (N = 1e5: 17.4 ms vs 21.8 ms at 128 levels), 24 columns per lane
// and 256 levels beyond (N = 1e6: 360 ms vs 375 ms); the right D columns of a
// warp's window are its ghost zone
constexpr int TREE_D = 256;  // levels per band (both shapes)
constexpr int TREE_THREADS = 128;

struct TreeConsts {
    double S0, K, K2, h, pu, pd, d, c0;
    int kind;
    int euro;  // European: no early exercise (NEXT #3)
};

__device__ __forceinline__ double max_nonneg(double x, double c) {  // max(x, c) for c >= +0
    return __longlong_as_double(max(__double_as_longlong(x), __double_as_longlong(c)));
}

// exercise state of column j at level t: put/call X = +-(K - S); bull: X = S
__device__ __forceinline__ double exercise_state(const TreeConsts& c, int t, int64_t j) {
    const double S = c.S0 * exp(c.h * (double)((int64_t)t - 2 * j));
    if (c.kind == KIND_PUT) return c.K - S;
    if (c.kind == KIND_CALL) return S - c.K;
    return S;
}
__device__ __forceinline__ double exercise_value(const TreeConsts& c, double X) {
    if (c.kind == KIND_BULL) return fmin(fmax(X - c.K, 0.0), c.K2 - c.K);
    return X;
}

// leaves: V_N(j) = max(P(S_{N,j}), 0) for j in [j0, j0 + n)
__global__ void tree_leaves_kernel(TreeConsts c, int N, int64_t j0, int64_t n, double* v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    v[i] = fmax(exercise_value(c, exercise_state(c, N, j0 + i)), 0.0);
}

// one band: levels t_top-1 .. t_top-D'; vin holds level t_top for columns
// [jin0, jin0 + nin); vout receives level t_top - D' for [jout0, jout0 + nout)
template <int TREE_M, int KIND, bool EURO>
__global__ void __launch_bounds__(TREE_THREADS) tree_band_kernel(TreeConsts c, int t_top, int Dp,
                                                                 const double* __restrict__ vin, int64_t jin0,
                                                                 int64_t nin, double* __restrict__ vout,
                                                                 int64_t jout0, int64_t nout) {
    constexpr int TREE_W = 32 * TREE_M - TREE_D;  // output columns per warp
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t jw = jout0 + w * TREE_W;
    if (jw >= jout0 + nout) return;  // warp-uniform
    double V[TREE_M], X[TREE_M];
#pragma unroll
    for (int q = 0; q < TREE_M; ++q) {
        const int64_t j = jw + lane * TREE_M + q;
        const int64_t i = j - jin0;
        V[q] = (i < nin) ? vin[i] : 0.0;  // beyond the window: ghost columns, never read back
        X[q] = exercise_state(c, t_top, j);
    }
    for (int l = 0; l < Dp; ++l) {
        const double nb = __shfl_down_sync(0xffffffffu, V[0], 1);
#pragma unroll
        for (int q = 0; q < TREE_M; ++q) {
            const double vn = (q + 1 < TREE_M) ? V[q + 1] : nb;
            double ex;
            if (KIND == KIND_BULL) {
                X[q] *= c.d;
                ex = fmin(fmax(X[q] - c.K, 0.0), c.K2 - c.K);
            } else {
                X[q] = fma(c.d, X[q], c.c0);
                ex = X[q];
            }
            const double cont = fma(c.pu, V[q], c.pd * vn);
            V[q] = EURO ? cont : max_nonneg(ex, cont);
        }
    }
#pragma unroll
    for (int q = 0; q < TREE_M; ++q) {
        const int64_t off = (int64_t)lane * TREE_M + q;
        const int64_t j = jw + off;
        if (off < TREE_W && j < jout0 + nout) vout[j - jout0] = V[q];
    }
}

// ---------------------------------------------------------------------------
// Wavefront kernel (one GPU): the same bands as tree_band_kernel, but ONE
// cooperative launch for the whole tree.  Warp w owns output slot w (columns
// [w W, (w+1) W), W = 32 M - D) at every band; its window at band b is slots w
// and w+1 of band b-1's output (the dependency cone of D levels).
// Instead of a launch boundary (and a window copy) per band, warp w waits on
// two progress counters: slot w+1 has published band b-1 (its producer) and
// slot w-1 has finished band b-1 (the last reader of the buffer slot w is
// about to overwrite: two level buffers, ping-pong by band parity).  Bands of
// different slots overlap in a wavefront; warps right of the level's width
// exit.  All warps must be co-resident (cooperative launch; the host falls back
// to one launch per band when they are not).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int TREE_M, int TD, int KIND, bool EURO, bool SCALED>
__global__ void __launch_bounds__(TREE_THREADS) tree_wave_kernel(TreeConsts c, int N, double* __restrict__ buf0,
                                                                 double* __restrict__ buf1, int* __restrict__ prog,
                                                                 int nslots) {
    constexpr int TW = 32 * TREE_M - TD;  // output columns per slot
    static_assert(TD <= TW, "the window of a slot spans slots w and w+1 only");
    static_assert(!SCALED || KIND != KIND_BULL, "the scaled recursion is for puts and calls");
    const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= nslots) return;  // warp-uniform
    const int64_t j0 = (int64_t)w * TW;
    double V[TREE_M], X[TREE_M];
    int b = 0;
    for (int t_top = N; t_top > 0; ++b) {
        const int Dp = min(TD, t_top);
        const int t_bot = t_top - Dp;
        if (j0 > t_bot) break;  // the output level has t_bot + 1 columns: this slot is done
        const double* vin = (b & 1) ? buf1 : buf0;
        double* vout = (b & 1) ? buf0 : buf1;
        if (b > 0) {
            if (lane == 0) {
                // producer: slot w+1 was active at band b-1 iff its first column <= t_top
                if (w + 1 < nslots && (int64_t)(w + 1) * TW <= t_top)
                    while (ld_acquire(prog + w + 1) < b) __nanosleep(16);
                if (w > 0)
                    while (ld_acquire(prog + w - 1) < b) __nanosleep(16);
            }
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < TREE_M; ++q) {
            const int64_t j = j0 + lane * TREE_M + q;
            X[q] = exercise_state(c, t_top, j);
            if (b == 0) V[q] = fmax(exercise_value(c, X[q]), 0.0);  // leaves (t = N)
            else V[q] = (j <= t_top) ? __ldcg(vin + j) : 0.0;  // beyond the level: ghost columns, never read back
        }
        double scale = 1.0;  // SCALED: V = scale * U after the band
        if (SCALED) {
            // U_t = V_t / pd^(t_top - t):  U_t(j) = max(E_t(j) / pd^(t_top - t), a U_{t+1}(j) + U_{t+1}(j+1)),
            // a = pu / pd -- one DFMA per node on the level-to-level chain; the
            // scaled exercise value follows Es_t = (d / pd) Es_{t+1} + c0 / pd^(t_top - t)
            const double a = c.pu / c.pd, dr = c.d / c.pd, ipd = 1.0 / c.pd;
            double g = c.c0;
            for (int l = 0; l < Dp; ++l) {
                const double nb = __shfl_down_sync(0xffffffffu, V[0], 1);
                g *= ipd;
                scale *= c.pd;
#pragma unroll
                for (int q = 0; q < TREE_M; ++q) {
                    const double vn = (q + 1 < TREE_M) ? V[q + 1] : nb;
                    X[q] = fma(dr, X[q], g);
                    const double cont = fma(a, V[q], vn);
                    V[q] = EURO ? cont : max_nonneg(X[q], cont);
                }
            }
        } else {
            for (int l = 0; l < Dp; ++l) {
                const double nb = __shfl_down_sync(0xffffffffu, V[0], 1);
#pragma unroll
                for (int q = 0; q < TREE_M; ++q) {
                    const double vn = (q + 1 < TREE_M) ? V[q + 1] : nb;
                    double ex;
                    if (KIND == KIND_BULL) {
                        X[q] *= c.d;
                        ex = fmin(fmax(X[q] - c.K, 0.0), c.K2 - c.K);
                    } else {
                        X[q] = fma(c.d, X[q], c.c0);
                        ex = X[q];
                    }
                    const double cont = fma(c.pu, V[q], c.pd * vn);
                    V[q] = EURO ? cont : max_nonneg(ex, cont);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < TREE_M; ++q) {
            const int off = lane * TREE_M + q;
            const int64_t j = j0 + off;
            if (off < TW && j <= t_bot) __stcg(vout + j, SCALED ? V[q] * scale : V[q]);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(prog + w, b + 1);
        t_top = t_bot;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int tree_consts(const amtc_params* p, int N, const amtc_payoff* pay, TreeConsts& c) {
    if (!p || !pay || (pay->flags & ~7u) || N < 1) return STATUS_EINVAL;  // cost-at-t0: no effect at k = 0
    if ((pay->flags & 2u) && pay->kind == KIND_BULL) return STATUS_EINVAL;  // AMTC_CASH: put / call only
    c.euro = (pay->flags & 1u) ? 1 : 0;  // AMTC_EUROPEAN (cash settlement: the same CRR value, A.1)
    if (!(p->S0 > 0.0) || !(p->T > 0.0) || !(p->sigma > 0.0) || !std::isfinite(p->R)) return STATUS_EINVAL;
    c.kind = pay->kind;
    c.S0 = p->S0;
    c.K = pay->K;
    c.K2 = pay->K2;
    if (c.kind != KIND_PUT && c.kind != KIND_CALL && c.kind != KIND_BULL) return STATUS_EINVAL;
    if (c.kind != KIND_BULL && !(c.K > 0.0)) return STATUS_EINVAL;
    if (c.kind == KIND_BULL && !(c.K < c.K2)) return STATUS_EINVAL;
    c.h = p->sigma * std::sqrt(p->T / (double)N);
    const double rho = p->R * p->T / (double)N;
    if (!(rho < c.h && -c.h < rho)) return STATUS_EARBITRAGE;  // d < r < u
    const double u = std::exp(c.h), r = std::exp(rho);
    c.d = 1.0 / u;
    const double pr = (r - c.d) / (u - c.d);  // risk-neutral probability
    c.pu = pr / r;
    c.pd = (1.0 - pr) / r;
    c.c0 = (c.kind == KIND_PUT) ? c.K * (1.0 - c.d) : -c.K * (1.0 - c.d);
    return STATUS_OK;
}

static void launch_leaves(const TreeConsts& c, int N, int64_t j0, int64_t n, double* v, cudaStream_t s) {
    if (n <= 0) return;
    tree_leaves_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c, N, j0, n, v);
    note_launch();
}

template <int M>
static void launch_band_m(const TreeConsts& c, int t_top, int Dp, const double* vin, int64_t jin0, int64_t nin,
                          double* vout, int64_t jout0, int64_t nout, cudaStream_t s) {
    constexpr int W = 32 * M - TREE_D;
    const int64_t warps = (nout + W - 1) / W;
    const unsigned blocks = (unsigned)((warps * 32 + TREE_THREADS - 1) / TREE_THREADS);
#define AMTC_BAND(K, E) \
    tree_band_kernel<M, K, E><<<blocks, TREE_THREADS, 0, s>>>(c, t_top, Dp, vin, jin0, nin, vout, jout0, nout)
    if (c.euro) {
        if (c.kind == KIND_PUT) AMTC_BAND(KIND_PUT, true);
        else if (c.kind == KIND_CALL) AMTC_BAND(KIND_CALL, true);
        else AMTC_BAND(KIND_BULL, true);
    } else {
        if (c.kind == KIND_PUT) AMTC_BAND(KIND_PUT, false);
        else if (c.kind == KIND_CALL) AMTC_BAND(KIND_CALL, false);
        else AMTC_BAND(KIND_BULL, false);
    }
#undef AMTC_BAND
}

static void launch_band(const TreeConsts& c, int N, int t_top, int Dp, const double* vin, int64_t jin0, int64_t nin,
                        double* vout, int64_t jout0, int64_t nout, cudaStream_t s) {
    if (nout <= 0) return;
    if (N <= 300000) launch_band_m<16>(c, t_top, Dp, vin, jin0, nin, vout, jout0, nout, s);
    else launch_band_m<24>(c, t_top, Dp, vin, jin0, nin, vout, jout0, nout, s);
    note_launch();
}

// grow-only device buffers of this translation unit (per device, mutex-guarded)
struct TreeBufs {
    std::mutex mu;
    double* p[3] = {nullptr, nullptr, nullptr};
    size_t n = 0;
    double* h_pinned = nullptr;
    cudaError_t ensure(size_t want) {
        if (want <= n) return cudaSuccess;
        for (auto& q : p) {
            if (q) cudaFree(q);
            q = nullptr;
        }
        n = 0;
        for (auto& q : p) {
            cudaError_t e = cudaMalloc(&q, want * sizeof(double));
            if (e != cudaSuccess) return e;
        }
        if (!h_pinned) {
            cudaError_t e = cudaMallocHost(&h_pinned, sizeof(double));
            if (e != cudaSuccess) return e;
        }
        n = want;
        return cudaSuccess;
    }
};
static TreeBufs* tree_bufs() {
    static std::mutex mu;
    static std::vector<TreeBufs*> v;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if ((int)v.size() <= dev) v.resize(dev + 1, nullptr);
    if (!v[dev]) v[dev] = new TreeBufs();
    return v[dev];
}

// rank g's columns of a level of width w over n ranks: [a_g, a_{g+1}),
// a_g = ceil(g w / n) (rank 0 keeps the root column)
// Processor reduction: a level of w columns is spread over
// n_act = clamp(w / TREE_MIN_COLS, 1, n) ranks only -- small levels near the root
// stay on rank 0 and the rest drop out instead of exchanging halos for a few
// columns each.  Rank g < n_act owns [ceil(g w / n_act), ceil((g+1) w / n_act)).
constexpr int64_t TREE_MIN_COLS = 4096;

static thread_local std::string t_err;
static int cuda_err(cudaError_t e, const char* what) {
    t_err = std::string(what) + ": " + cudaGetErrorString(e);
    return STATUS_ECUDA;
}

// The exchange plan of one band (host only; exported as amtc_tree_band_plan so
// the multi-rank CPU test drives the library's own plan): rank `rank`'s input
// columns [own_lo, own_hi) at t_top, its output columns [new_lo, new_hi) at
// t_top - Dp, its window [win_lo, win_hi) at t_top (new range + Dp halo columns
// from the right: the dependency cone) and, per peer g, the columns
// [send[2g], send[2g+1]) of level t_top it sends to g and [recv[2g],
// recv[2g+1]) it receives from g (empty ranges: lo == hi).  min_cols: the
// processor-reduction threshold (columns per active rank).
struct BandPlan {
    int t_top, Dp;
    int64_t own_lo, own_hi, new_lo, new_hi, win_lo, win_hi;
};
static void band_plan(int t_top, int D, int rank, int nranks, int64_t mc, BandPlan& P, int64_t* send, int64_t* recv) {
    auto split = [&](int64_t w, int g) {
        const int64_t na = std::max<int64_t>(1, std::min<int64_t>(nranks, w / mc));
        return g >= na ? w : (g * w + na - 1) / na;
    };
    P.t_top = t_top;
    P.Dp = std::min(D, t_top);
    const int64_t w1 = t_top + 1, w0 = t_top - P.Dp + 1;
    auto need = [&](int g, int64_t& lo, int64_t& hi) {
        const int64_t a0 = split(w0, g), b0 = split(w0, g + 1);
        lo = a0;
        hi = (b0 > a0) ? std::min(b0 + P.Dp, w1) : a0;
    };
    P.own_lo = split(w1, rank);
    P.own_hi = split(w1, rank + 1);
    P.new_lo = split(w0, rank);
    P.new_hi = split(w0, rank + 1);
    need(rank, P.win_lo, P.win_hi);
    for (int g = 0; g < nranks; ++g) {
        send[2 * g] = send[2 * g + 1] = recv[2 * g] = recv[2 * g + 1] = 0;
        if (g == rank) continue;
        int64_t lo, hi;
        need(g, lo, hi);
        const int64_t s0 = std::max(lo, P.own_lo), s1 = std::min(hi, P.own_hi);
        if (s1 > s0) { send[2 * g] = s0; send[2 * g + 1] = s1; }
        const int64_t ga = split(w1, g), gb = split(w1, g + 1);
        const int64_t r0 = std::max(P.win_lo, ga), r1 = std::min(P.win_hi, gb);
        if (r1 > r0) { recv[2 * g] = r0; recv[2 * g + 1] = r1; }
    }
}
// columns of each of the three level buffers: the widest own range or window
// of any band (checked against every band by the CPU test through
// amtc_tree_band_plan): ceil((N+1)/n) while every rank is active, up to
// 2 min_cols - 1 on rank 0 while fewer are (processor reduction), + the halo
static int64_t tree_cap(int N, int nranks, int D, int64_t mc) {
    return std::max<int64_t>((N + 1 + nranks - 1) / nranks, 2 * mc) + D + 64;
}

// testing hook amtc_debug_set_tree_shape: 0 auto, 1 one launch per band,
// 2..5 the wavefront kernel with (M, D) = (16, 256), (8, 128), (12, 128), (8, 64)
static std::atomic<int> g_tree_shape{0};

template <int M, int TD>
static cudaError_t wave_launch(const TreeConsts& c, int N, double* b0, double* b1, int* prog, int& nslots,
                               cudaStream_t s, bool scaled) {
    constexpr int TW = 32 * M - TD;
    nslots = (N + 1 + TW - 1) / TW;
    const unsigned blocks = (unsigned)((nslots * 32 + TREE_THREADS - 1) / TREE_THREADS);
    void* fn = nullptr;
#define AMTC_WAVE_FN(K, E) fn = (K != KIND_BULL && scaled) ? (void*)tree_wave_kernel<M, TD, (K == KIND_BULL ? KIND_PUT : K), E, true> \
                                                           : (void*)tree_wave_kernel<M, TD, K, E, false>
    if (c.euro) {
        if (c.kind == KIND_PUT) AMTC_WAVE_FN(KIND_PUT, true);
        else if (c.kind == KIND_CALL) AMTC_WAVE_FN(KIND_CALL, true);
        else AMTC_WAVE_FN(KIND_BULL, true);
    } else {
        if (c.kind == KIND_PUT) AMTC_WAVE_FN(KIND_PUT, false);
        else if (c.kind == KIND_CALL) AMTC_WAVE_FN(KIND_CALL, false);
        else AMTC_WAVE_FN(KIND_BULL, false);
    }
#undef AMTC_WAVE_FN
    cudaError_t e = cudaMemsetAsync(prog, 0, sizeof(int) * (size_t)nslots, s);
    if (e != cudaSuccess) return e;
    TreeConsts cc = c;
    int n = N, ns = nslots;
    void* args[] = {&cc, &n, &b0, &b1, &prog, &ns};
    // cooperative: every warp co-resident (the progress waits need it) or an error
    e = cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(TREE_THREADS), args, 0, s);
    if (e == cudaSuccess) note_launch();
    return e;
}

// one GPU: the whole tree in one wavefront launch; false if it does not fit
// (too many slots to be co-resident): the caller runs the banded path
static bool tree_wave(const TreeConsts& c, int N, TreeBufs* B, double* price, cudaStream_t s, int& st) {
    int shape = g_tree_shape.load();
    if (shape == 1) return false;
    if (shape == 0) shape = (N <= 300000) ? 3 : 2;
    int nslots = 0;
    double* const b0 = B->p[0];
    double* const b1 = B->p[1];
    int* const prog = reinterpret_cast<int*>(B->p[2]);
    cudaError_t e;
    int D = 0;
    const bool scaled = shape >= 10;
    switch (shape % 10) {
        case 2: e = wave_launch<16, 256>(c, N, b0, b1, prog, nslots, s, scaled); D = 256; break;
        case 4: e = wave_launch<12, 128>(c, N, b0, b1, prog, nslots, s, scaled); D = 128; break;
        case 5: e = wave_launch<8, 64>(c, N, b0, b1, prog, nslots, s, scaled); D = 64; break;
        case 6: e = wave_launch<4, 64>(c, N, b0, b1, prog, nslots, s, scaled); D = 64; break;
        case 7: e = wave_launch<6, 96>(c, N, b0, b1, prog, nslots, s, scaled); D = 96; break;
        case 8: e = wave_launch<4, 32>(c, N, b0, b1, prog, nslots, s, scaled); D = 32; break;
        default: e = wave_launch<8, 128>(c, N, b0, b1, prog, nslots, s, scaled); D = 128; break;
    }
    if (e == cudaErrorCooperativeLaunchTooLarge) {
        cudaGetLastError();  // clear
        return false;
    }
    if (e != cudaSuccess) { st = cuda_err(e, "tree wave launch"); return true; }
    // the last band (index nb - 1) writes level 0 into buf1 (nb - 1 even) or buf0
    const int nb = (N + D - 1) / D;
    const double* root = ((nb - 1) & 1) ? b0 : b1;
    e = cudaMemcpyAsync(B->h_pinned, root, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) { st = cuda_err(e, "tree wave"); return true; }
    *price = *B->h_pinned;
    st = STATUS_OK;
    return true;
}

// the whole tree, ranks 0..n-1 of comm (comm == nullptr: one GPU, no NCCL)
static int tree_run(const TreeConsts& c, int N, ncclComm_t comm, int rank, int nranks, double* price,
                    cudaStream_t s) {
    TreeBufs* B = tree_bufs();
    std::lock_guard<std::mutex> guard(B->mu);
    const int64_t cap = tree_cap(N, nranks, TREE_D, TREE_MIN_COLS);
    cudaError_t e = B->ensure((size_t)cap);
    if (e != cudaSuccess) return cuda_err(e, "tree buffers");
    if (!comm && nranks == 1) {
        int st = STATUS_OK;
        if (tree_wave(c, N, B, price, s, st)) return st;
    }
    double* cur = B->p[0];   // own columns of the current level
    double* win = B->p[1];   // input window of the band
    double* nxt = B->p[2];   // own columns of the next level
    std::vector<int64_t> snd(2 * (size_t)nranks), rcv(2 * (size_t)nranks);
    // leaves (t = N), own range
    BandPlan P;
    band_plan(N, TREE_D, rank, nranks, TREE_MIN_COLS, P, snd.data(), rcv.data());
    launch_leaves(c, N, P.own_lo, P.own_hi - P.own_lo, cur, s);
    for (int t_top = N; t_top > 0;) {
        band_plan(t_top, TREE_D, rank, nranks, TREE_MIN_COLS, P, snd.data(), rcv.data());
        const int Dp = P.Dp;
        const int t_bot = t_top - Dp;
        const int64_t a = P.own_lo, b = P.own_hi, my_lo = P.win_lo, my_hi = P.win_hi;
        if (b - a > cap || my_hi - my_lo > cap || P.new_hi - P.new_lo > cap) {  // cannot happen (tree_cap)
            t_err = "sharded tree: rank range exceeds its buffers";
            return STATUS_EINVAL;
        }
        // gather the window: intersections of owners' ranges with windows
        if (comm) {
            if (ncclGroupStart() != ncclSuccess) return STATUS_ENCCL;
        }
        for (int g = 0; g < nranks; ++g) {
            if (g == rank) continue;
            const int64_t s0 = snd[2 * g], s1 = snd[2 * g + 1], r0 = rcv[2 * g], r1 = rcv[2 * g + 1];
            if (s1 > s0 && ncclSend(cur + (s0 - a), (size_t)(s1 - s0), ncclDouble, g, comm, s) != ncclSuccess)
                return STATUS_ENCCL;
            if (r1 > r0 && ncclRecv(win + (r0 - my_lo), (size_t)(r1 - r0), ncclDouble, g, comm, s) != ncclSuccess)
                return STATUS_ENCCL;
        }
        if (comm) {
            if (ncclGroupEnd() != ncclSuccess) return STATUS_ENCCL;
        }
        {
            const int64_t x0 = std::max(my_lo, a), x1 = std::min(my_hi, b);
            if (x1 > x0) {
                e = cudaMemcpyAsync(win + (x0 - my_lo), cur + (x0 - a), sizeof(double) * (x1 - x0),
                                    cudaMemcpyDeviceToDevice, s);
                if (e != cudaSuccess) return cuda_err(e, "window copy");
            }
        }
        launch_band(c, N, t_top, Dp, win, my_lo, my_hi - my_lo, nxt, P.new_lo, P.new_hi - P.new_lo, s);
        std::swap(cur, nxt);
        t_top = t_bot;
    }
    // the root column belongs to rank 0; share it
    if (comm) {
        if (ncclBroadcast(cur, cur, 1, ncclDouble, 0, comm, s) != ncclSuccess) return STATUS_ENCCL;
    }
    e = cudaMemcpyAsync(B->h_pinned, cur, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_err(e, "root copy");
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_err(e, "tree sync");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_err(e, "tree kernels");
    *price = *B->h_pinned;
    return STATUS_OK;
}

}  // namespace amtc

using namespace amtc;

extern "C" {

int amtc_price_crr_tree(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double* price,
                        void* cuda_stream) {
    try {
        if (!price) return STATUS_EINVAL;
        *price = NAN;
        TreeConsts c;
        const int st = tree_consts(params, N, payoff, c);
        if (st) return st;
        return tree_run(c, N, nullptr, 0, 1, price, static_cast<cudaStream_t>(cuda_stream));
    } catch (...) {
        return STATUS_ECUDA;
    }
}

int amtc_comm_unique_id(unsigned char id[128]) {
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return STATUS_ENCCL;
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
    for (int i = 0; i < 128; ++i) id[i] = (unsigned char)u.internal[i];
    return STATUS_OK;
}

int amtc_comm_init(const unsigned char id[128], int nranks, int rank, void** comm_out) {
    if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return STATUS_EINVAL;
    ncclUniqueId u;
    for (int i = 0; i < 128; ++i) u.internal[i] = (char)id[i];
    ncclComm_t comm;
    if (ncclCommInitRank(&comm, nranks, u, rank) != ncclSuccess) return STATUS_ENCCL;
    *comm_out = comm;
    return STATUS_OK;
}

int amtc_comm_destroy(void* comm) {
    if (!comm) return STATUS_EINVAL;
    return ncclCommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? STATUS_OK : STATUS_ENCCL;
}

void amtc_debug_set_tree_shape(int shape) { g_tree_shape.store(shape); }

int amtc_tree_band_plan(int32_t N, int nranks, int rank, int32_t band, int32_t D, int64_t min_cols,
                        amtc_band* out, int64_t* send, int64_t* recv, int32_t* n_bands) {
    if (N < 1 || nranks < 1 || rank < 0 || rank >= nranks || D < 0 || min_cols < 0) return STATUS_EINVAL;
    if (D == 0) D = TREE_D;
    if (min_cols == 0) min_cols = TREE_MIN_COLS;
    const int32_t nb = (N + D - 1) / D;
    if (n_bands) *n_bands = nb;
    if (band < 0 || band >= nb || !out || !send || !recv) return (band == -1 && n_bands) ? STATUS_OK : STATUS_EINVAL;
    BandPlan P;
    band_plan(N - band * D, D, rank, nranks, min_cols, P, send, recv);
    out->t_top = P.t_top;
    out->Dp = P.Dp;
    out->own_lo = P.own_lo;
    out->own_hi = P.own_hi;
    out->new_lo = P.new_lo;
    out->new_hi = P.new_hi;
    out->win_lo = P.win_lo;
    out->win_hi = P.win_hi;
    out->cap = tree_cap(N, nranks, D, min_cols);
    return STATUS_OK;
}

int amtc_price_tree_sharded(const amtc_params* params, int32_t N, const amtc_payoff* payoff, double k,
                            void* nccl_comm, int rank, int nranks, amtc_quote* out, void* cuda_stream) {
    try {
        if (!out) return STATUS_EINVAL;
        out->ask = out->bid = NAN;
        out->max_bp = 0;
        out->status = STATUS_EINVAL;
        if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_comm)) return STATUS_EINVAL;
        if (!(k >= 0.0 && k < 1.0)) return STATUS_EINVAL;
        if (k > 0.0) {
            // the transaction-cost tree: strips partitioned over the ranks, the
            // boundary carry column read from the next GPU (amtc_capi.cu)
            if (nranks == 1 && !nccl_comm) {
                *out = amtc_price_american_tc(params, N, payoff, k);
                return out->status;
            }
            if (!params || !payoff) return STATUS_EINVAL;
            if (N < 64) {  // too small to shard: every rank prices it alone
                *out = amtc_price_american_tc(params, N, payoff, k);
                return out->status;
            }
            const int st = tc_tree_sharded(params, N, payoff, k, nccl_comm, rank, nranks, out,
                                           static_cast<cudaStream_t>(cuda_stream));
            out->status = st;
            return st;
        }
        TreeConsts c;
        int st = tree_consts(params, N, payoff, c);
        if (st) { out->status = st; return st; }
        double price = NAN;
        st = tree_run(c, N, static_cast<ncclComm_t>(nccl_comm), rank, nranks, &price,
                      static_cast<cudaStream_t>(cuda_stream));
        out->status = st;
        if (!st) {
            out->ask = price;  // k = 0: ask = bid = the CRR price (derived A.1)
            out->bid = price;
            out->max_bp = 1;
        }
        return st;
    } catch (...) {
        return STATUS_ECUDA;
    }
}

}  // extern "C"
