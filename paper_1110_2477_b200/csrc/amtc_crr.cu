// amtc_crr.cu -- k = 0 (frictionless) batched American CRR pricing
// (Appendix: no extra level, scalar max).
//
//   V_N(j) = max(P(S_{N,j}), 0),
//   V_t(j) = max(P(S_{t,j}), p_u V_{t+1}(j) + p_d V_{t+1}(j+1)),
//   p_u = p / r, p_d = (1-p)/r, p = (r-d)/(u-d).
//
// One warp per tree; the level lives in registers.  Layout: lane l holds, for
// every slot c, the M = 4 consecutive nodes j = (32 c + l) M + q, q = 0..3
// (blocked-cyclic).  The down child of a lane's last node is the first node of
// lane l+1 (same slot), or of lane 0 in slot c+1 for lane 31: one 64-bit
// shuffle per slot per level, amortised over M nodes.  As the level shrinks
// whole slots retire (the slot loop is warp-uniform), so no rebalancing is
// needed and at most one slot per level is partially idle.
//
// The exercise value is carried incrementally: S_{t,j} = d S_{t+1,j}, so for
// the put X = K - S obeys X_t = d X_{t+1} + K(1-d) (one DFMA), for the call
// X_t = d X_{t+1} - K(1-d); the bull spread keeps S and clamps.
// FP64 per node-update: DFMA (X) + DMUL + DFMA (continuation); the max runs on the integer ALU.
#include <cuda_runtime.h>

#include <algorithm>

#include "amtc_internal.cuh"

namespace amtc {

constexpr int CRR_M = 4;

// max(x, c) for c >= +0 and min(a, b) for a, b >= +0 as signed 64-bit integer
// max / min of the bit patterns (IEEE order of non-negative doubles is the
// integer order; a negative x has a negative pattern): integer-ALU work instead
// of the FP64 pipe's DMNMX, which issues at 1/4.5 of the DFMA rate on B200
// (profiles/r01_fp64_peak.json).  Every V is >= +0 (max with a continuation
// value p_u V + p_d V' of non-negative values).
__device__ __forceinline__ double max_nonneg(double x, double c) {
    return __longlong_as_double(max(__double_as_longlong(x), __double_as_longlong(c)));
}
__device__ __forceinline__ double min_nonneg(double a, double b) {
    return __longlong_as_double(min(__double_as_longlong(a), __double_as_longlong(b)));
}
constexpr int CRR_THREADS = 128;

// payoff at the leaves: put (K - S)+, call (S - K)+, bull clamp
template <int KIND>
__device__ __forceinline__ double crr_payoff(double S, double K, double K2) {
    if (KIND == KIND_PUT) return fmax(K - S, 0.0);
    if (KIND == KIND_CALL) return fmax(S - K, 0.0);
    return fmin(fmax(S - K, 0.0), K2 - K);
}

// The registers hold nodes j = 0 .. 128 C - 1 of the level; C = ceil(N / 128),
// so the leaf j = N may fall outside them (N = 1024: 8 slots, not 9) -- it is
// only read once, as the down child of node N-1 at t = N-1, and enters as a
// scalar through the slot-shift shuffle.
template <int C, int KIND, bool EURO>
__device__ __forceinline__ double crr_tree(int lane, int N, double S0, double K, double K2, double h, double rho) {
    const double u = exp(h), d = 1.0 / u, r = exp(rho);
    const double p = (r - d) / (u - d);
    const double pu = p / r, pd = (1.0 - p) / r;
    const double c0 = (KIND == KIND_PUT) ? K * (1.0 - d) : -K * (1.0 - d);

    double V[C][CRR_M], X[C][CRR_M];
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
        for (int q = 0; q < CRR_M; ++q) {
            const int j = (32 * c + lane) * CRR_M + q;
            const double S = S0 * exp(h * (double)(N - 2 * j));
            double x;
            if (KIND == KIND_PUT) x = K - S;
            else if (KIND == KIND_CALL) x = S - K;
            else x = S;  // bull: X holds S
            X[c][q] = x;
            V[c][q] = crr_payoff<KIND>(S, K, K2);
        }
    }
    // the leaf j = N when the slots end at j = N - 1
    double leafN = (N == 32 * CRR_M * C) ? crr_payoff<KIND>(S0 * exp(-h * (double)N), K, K2) : 0.0;
    for (int t = N - 1; t >= 0; --t) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (32 * c * CRR_M > t) break;  // warp-uniform: slot c holds no live node
            const double send = (lane == 0) ? ((c + 1 < C) ? V[c + 1][0] : leafN) : V[c][0];
            const double nb = __shfl_sync(0xffffffffu, send, (lane + 1) & 31);
#pragma unroll
            for (int q = 0; q < CRR_M; ++q) {
                const double vn = (q + 1 < CRR_M) ? V[c][q + 1] : nb;
                double ex;
                if (KIND == KIND_BULL) {
                    X[c][q] *= d;
                    ex = min_nonneg(max_nonneg(X[c][q] - K, 0.0), K2 - K);
                } else {
                    X[c][q] = fma(d, X[c][q], c0);
                    ex = X[c][q];
                }
                const double cont = fma(pu, V[c][q], pd * vn);
                V[c][q] = EURO ? cont : max_nonneg(ex, cont);  // European: no early exercise (NEXT #3)
            }
        }
        leafN = 0.0;
    }
    return V[0][0];
}

// Large N (beyond the register-resident level): the warp sweeps the tree in
// vertical strips of 32 * SM columns, right to left (the TC solver's strip
// order; region-B dependency P:164-166).  Lane l owns columns
// j0 + l SM .. j0 + l SM + SM - 1 of strip [j0, j0 + 32 SM) from the leaves
// (t = N) down to t = j0; the down child of lane 31's last column is column
// j0 + 32 SM of the strip to the right, read from the carry buffer that strip
// wrote at every level (prefetched one level ahead).  Exact work: every node
// (t, j), j <= t, is updated once (plus at most one partially live strip per
// level).  cbuf: 2 (N + 2) doubles per warp (ping-pong by strip parity).
constexpr int CRR_SM = 16;
template <int KIND, bool EURO>
__device__ double crr_strip_tree(int lane, int N, double S0, double K, double K2, double h, double rho,
                                 double* cbuf) {
    constexpr int SM = CRR_SM, WD = 32 * CRR_SM;
    const double u = exp(h), d = 1.0 / u, r = exp(rho);
    const double p = (r - d) / (u - d);
    const double pu = p / r, pd = (1.0 - p) / r;
    const double c0 = (KIND == KIND_PUT) ? K * (1.0 - d) : -K * (1.0 - d);
    const int ns = N / WD + 1;  // strips covering columns 0..N
    double V[SM], X[SM];
    for (int s = ns - 1; s >= 0; --s) {
        const int j0 = s * WD;
        double* const cout = cbuf + (size_t)(s & 1) * (N + 2);
        const double* const cin = cbuf + (size_t)((s + 1) & 1) * (N + 2);
        const bool has_right = s < ns - 1;
#pragma unroll
        for (int q = 0; q < SM; ++q) {  // leaves t = N
            const int j = j0 + lane * SM + q;
            const double S = S0 * exp(h * (double)(N - 2 * j));
            if (KIND == KIND_PUT) X[q] = K - S;
            else if (KIND == KIND_CALL) X[q] = S - K;
            else X[q] = S;
            V[q] = crr_payoff<KIND>(S, K, K2);
        }
        if (s > 0 && lane == 0) cout[N] = V[0];
        // lane 31's down child of level t+1 (column j0 + WD), valid once t+1 >= j0 + WD
        double cr = (has_right && lane == 31 && N >= j0 + WD) ? cin[N] : 0.0;
        for (int t = N - 1; t >= j0; --t) {
            const double pre = (has_right && lane == 31 && t >= j0 + WD) ? cin[t] : 0.0;  // next level's
            double nb = __shfl_down_sync(0xffffffffu, V[0], 1);
            if (lane == 31) nb = cr;
#pragma unroll
            for (int q = 0; q < SM; ++q) {
                const double vn = (q + 1 < SM) ? V[q + 1] : nb;
                double ex;
                if (KIND == KIND_BULL) {
                    X[q] *= d;
                    ex = min_nonneg(max_nonneg(X[q] - K, 0.0), K2 - K);
                } else {
                    X[q] = fma(d, X[q], c0);
                    ex = X[q];
                }
                const double cont = fma(pu, V[q], pd * vn);
                V[q] = EURO ? cont : max_nonneg(ex, cont);
            }
            if (s > 0 && lane == 0) cout[t] = V[0];
            cr = pre;
        }
        __syncwarp();  // this strip's carry writes are visible to lane 31 in the next strip
    }
    return __shfl_sync(0xffffffffu, V[0], 0);
}

#ifndef AMTC_CRR_MINB
#define AMTC_CRR_MINB 1
#endif
// per-option validation (as the TC path's): NaN on failure
__device__ __forceinline__ bool crr_option(const BatchPtrs& in, int64_t w, int N, double& S0, double& K, double& K2,
                                           double& h, double& rho, int& kind, bool& euro) {
    S0 = in.S0[w]; K = in.K[w];
    const double T = in.T[w], sigma = in.sigma[w], R = in.R[w];
    K2 = in.K2 ? in.K2[w] : 0.0;
    kind = in.kind[w];
    const unsigned flags = in.flags ? in.flags[w] : 0u;
    euro = (flags & FLAG_EUROPEAN) != 0;  // cash settlement: the same CRR value (A.1)
    bool ok = (S0 > 0.0) && (T > 0.0) && (sigma > 0.0) && isfinite(R);
    ok = ok && !(flags & ~FLAG_ALL) && !((flags & FLAG_CASH) && kind == KIND_BULL);
    ok = ok && (kind == KIND_PUT || kind == KIND_CALL || kind == KIND_BULL);
    ok = ok && (kind == KIND_BULL ? (K < K2) : (K > 0.0));
    h = sigma * sqrt(T / (double)N);
    rho = R * T / (double)N;
    return ok && (rho < h) && (-h < rho);  // d < r < u
}

template <int C>
__global__ void __launch_bounds__(CRR_THREADS, AMTC_CRR_MINB) crr_kernel(BatchPtrs in, int64_t n, int N, double* out) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n) return;
    double S0, K, K2, h, rho;
    int kind;
    bool euro;
    double v = NAN;
    if (crr_option(in, w, N, S0, K, K2, h, rho, kind, euro)) {  // warp-uniform
        if (euro) {
            if (kind == KIND_PUT) v = crr_tree<C, KIND_PUT, true>(lane, N, S0, K, K2, h, rho);
            else if (kind == KIND_CALL) v = crr_tree<C, KIND_CALL, true>(lane, N, S0, K, K2, h, rho);
            else v = crr_tree<C, KIND_BULL, true>(lane, N, S0, K, K2, h, rho);
        } else {
            if (kind == KIND_PUT) v = crr_tree<C, KIND_PUT, false>(lane, N, S0, K, K2, h, rho);
            else if (kind == KIND_CALL) v = crr_tree<C, KIND_CALL, false>(lane, N, S0, K, K2, h, rho);
            else v = crr_tree<C, KIND_BULL, false>(lane, N, S0, K, K2, h, rho);
        }
    }
    if (lane == 0) out[w] = v;
}

// persistent warps: warp g prices options g, g + G, ... with its own carry buffer
__global__ void __launch_bounds__(CRR_THREADS) crr_strip_kernel(BatchPtrs in, int64_t n, int N, double* out,
                                                               double* ws) {
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t G = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    double* const cbuf = ws + (size_t)g * 2 * (N + 2);
    for (int64_t w = g; w < n; w += G) {
        double S0, K, K2, h, rho;
        int kind;
        bool euro;
        double v = NAN;
        if (crr_option(in, w, N, S0, K, K2, h, rho, kind, euro)) {
            if (euro) {
                if (kind == KIND_PUT) v = crr_strip_tree<KIND_PUT, true>(lane, N, S0, K, K2, h, rho, cbuf);
                else if (kind == KIND_CALL) v = crr_strip_tree<KIND_CALL, true>(lane, N, S0, K, K2, h, rho, cbuf);
                else v = crr_strip_tree<KIND_BULL, true>(lane, N, S0, K, K2, h, rho, cbuf);
            } else {
                if (kind == KIND_PUT) v = crr_strip_tree<KIND_PUT, false>(lane, N, S0, K, K2, h, rho, cbuf);
                else if (kind == KIND_CALL) v = crr_strip_tree<KIND_CALL, false>(lane, N, S0, K, K2, h, rho, cbuf);
                else v = crr_strip_tree<KIND_BULL, false>(lane, N, S0, K, K2, h, rho, cbuf);
            }
        }
        if (lane == 0) out[w] = v;
        __syncwarp();
    }
}

template <int C>
static void crr_launch_c(const BatchPtrs& in, int64_t n, int N, double* out, cudaStream_t s) {
    const int64_t threads = n * 32;
    const unsigned blocks = (unsigned)((threads + CRR_THREADS - 1) / CRR_THREADS);
    crr_kernel<C><<<blocks, CRR_THREADS, 0, s>>>(in, n, N, out);
    note_launch();
}

int crr_max_n() { return 32 * CRR_M * 9; }

int crr_launch(const BatchPtrs& in, int64_t n, int N, double* out, cudaStream_t s) {
    const int C = (N + 32 * CRR_M - 1) / (32 * CRR_M);  // the level t = N-1 holds N nodes
    switch (C) {
#define CASE(cc) \
    case cc: crr_launch_c<cc>(in, n, N, out, s); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
        default: return STATUS_EINVAL;
    }
    return STATUS_OK;
}

// resident warps of the strip kernel on this device (the persistent grid)
int64_t crr_strip_warps(int64_t n) {
    int dev = 0, sms = 0, b = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, crr_strip_kernel, CRR_THREADS, 0);
    const int64_t warps = (int64_t)std::max(sms, 1) * std::max(b, 1) * (CRR_THREADS / 32);
    const int64_t per = CRR_THREADS / 32;  // whole blocks: every launched warp owns a carry buffer
    return (std::min<int64_t>(warps, n) + per - 1) / per * per;
}
size_t crr_strip_ws_bytes(int N, int64_t warps) { return sizeof(double) * 2 * ((size_t)N + 2) * (size_t)warps; }

int crr_strip_launch(const BatchPtrs& in, int64_t n, int N, double* out, double* ws, int64_t warps,
                     cudaStream_t s) {
    const unsigned blocks = (unsigned)((warps * 32 + CRR_THREADS - 1) / CRR_THREADS);
    crr_strip_kernel<<<blocks, CRR_THREADS, 0, s>>>(in, n, N, out, ws);
    note_launch();
    return STATUS_OK;
}

}  // namespace amtc
