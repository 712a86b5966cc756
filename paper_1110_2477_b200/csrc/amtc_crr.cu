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
            V[c][q] = (KIND == KIND_BULL) ? fmin(fmax(S - K, 0.0), K2 - K) : fmax(x, 0.0);
        }
    }
    for (int t = N - 1; t >= 0; --t) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (32 * c * CRR_M > t) break;  // warp-uniform: slot c holds no live node
            const double send = (lane == 0) ? ((c + 1 < C) ? V[c + 1][0] : 0.0) : V[c][0];
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
    }
    return V[0][0];
}

#ifndef AMTC_CRR_MINB
#define AMTC_CRR_MINB 1
#endif
template <int C>
__global__ void __launch_bounds__(CRR_THREADS, AMTC_CRR_MINB) crr_kernel(BatchPtrs in, int64_t n, int N, double* out) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n) return;
    const double S0 = in.S0[w], K = in.K[w], T = in.T[w], sigma = in.sigma[w], R = in.R[w];
    const double K2 = in.K2 ? in.K2[w] : 0.0;
    const int kind = in.kind[w];
    const unsigned flags = in.flags ? in.flags[w] : 0u;
    const bool euro = (flags & FLAG_EUROPEAN) != 0;  // cash settlement: the same CRR value (A.1)
    bool ok = (S0 > 0.0) && (T > 0.0) && (sigma > 0.0) && isfinite(R);
    ok = ok && !(flags & ~FLAG_ALL) && !((flags & FLAG_CASH) && kind == KIND_BULL);
    ok = ok && (kind == KIND_PUT || kind == KIND_CALL || kind == KIND_BULL);
    ok = ok && (kind == KIND_BULL ? (K < K2) : (K > 0.0));
    const double h = sigma * sqrt(T / (double)N), rho = R * T / (double)N;
    ok = ok && (rho < h) && (-h < rho);  // d < r < u
    double v = NAN;
    if (ok) {  // warp-uniform
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

template <int C>
static void crr_launch_c(const BatchPtrs& in, int64_t n, int N, double* out, cudaStream_t s) {
    const int64_t threads = n * 32;
    const unsigned blocks = (unsigned)((threads + CRR_THREADS - 1) / CRR_THREADS);
    crr_kernel<C><<<blocks, CRR_THREADS, 0, s>>>(in, n, N, out);
    note_launch();
}

int crr_max_n() { return 32 * CRR_M * 9 - 1; }

int crr_launch(const BatchPtrs& in, int64_t n, int N, double* out, cudaStream_t s) {
    const int C = (N + 1 + 32 * CRR_M - 1) / (32 * CRR_M);
    switch (C) {
#define CASE(cc) \
    case cc: crr_launch_c<cc>(in, n, N, out, s); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
        default: return STATUS_EINVAL;
    }
    return STATUS_OK;
}

}  // namespace amtc
