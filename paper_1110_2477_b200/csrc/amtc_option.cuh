// amtc_option.cuh -- per-option model constants shared by the device code:
// validation (SURVEY 8(b) error conventions), CRR calibration and the
// payoff process.  Not part of the public C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cmath>

#include "amtc_internal.cuh"

namespace amtc {

struct OptionConsts {
    double S0, K, K2, k, h, rho;  // h = sigma sqrt(T/N) (u = e^h, d = 1/u), rho = R T / N (r = e^rho)
    int kind;
    unsigned flags;  // FLAG_EUROPEAN | FLAG_CASH
};

// Reads option i of the batch and validates it.  need_k = false reads k as 0
// (the frictionless CRR path).  Returns a STATUS_* code.
__device__ __forceinline__ int validate_option(const BatchPtrs& in, int64_t i, int N, bool need_k,
                                               OptionConsts& oc) {
    oc.S0 = in.S0[i];
    oc.K = in.K[i];
    oc.K2 = in.K2 ? in.K2[i] : 0.0;
    const double T = in.T[i], sigma = in.sigma[i], R = in.R[i];
    oc.k = (need_k && in.k) ? in.k[i] : 0.0;
    oc.kind = in.kind[i];
    oc.flags = in.flags ? in.flags[i] : 0u;
    if (!(oc.S0 > 0.0) || !(T > 0.0) || !(sigma > 0.0) || N < 1) return STATUS_EINVAL;
    if ((oc.flags & ~FLAG_ALL) || ((oc.flags & FLAG_CASH) && oc.kind == KIND_BULL)) return STATUS_EINVAL;
    if (!(oc.k >= 0.0 && oc.k < 1.0)) return STATUS_EINVAL;  // k in [0,1)
    if (oc.kind != KIND_PUT && oc.kind != KIND_CALL && oc.kind != KIND_BULL) return STATUS_EINVAL;
    if (oc.kind != KIND_BULL && !(oc.K > 0.0)) return STATUS_EINVAL;
    if (oc.kind == KIND_BULL && !(oc.K < oc.K2)) return STATUS_EINVAL;
    if (!isfinite(R)) return STATUS_EINVAL;
    oc.h = sigma * sqrt(T / (double)N);
    oc.rho = R * T / (double)N;
    // d < r < u  <=>  -h < rho < h  (risk-neutral p in (0,1))
    if (!(oc.rho < oc.h && -oc.h < oc.rho)) return STATUS_EARBITRAGE;
    return STATUS_OK;
}

// payoff process (xi, zeta) at stock price S: put (K, -1) physical;
// call (-K, +1) physical (reading A6); bull spread cash ((S-K)^+ - (S-K2)^+, 0)
// (cash-settled put / call, NEXT #3: ((K-S)^+, 0) / ((S-K)^+, 0))
__device__ __forceinline__ void option_payoff(const OptionConsts& oc, double S, double& xi, double& zeta) {
    if (oc.flags & FLAG_CASH) {
        xi = (oc.kind == KIND_PUT) ? fmax(oc.K - S, 0.0) : fmax(S - oc.K, 0.0);
        zeta = 0.0;
    } else if (oc.kind == KIND_PUT) { xi = oc.K; zeta = -1.0; }
    else if (oc.kind == KIND_CALL) { xi = -oc.K; zeta = 1.0; }
    else { xi = fmax(S - oc.K, 0.0) - fmax(S - oc.K2, 0.0); zeta = 0.0; }
}

}  // namespace amtc
