// amtc_root.cuh -- a6, the root t = 0 of the transaction-cost recursion, shared
// by the solver kernels (strip, light, full): no costs at t = 0, so
// v_0 is a line and ask / bid follow from the level-1 functions (lanes 0 and 1
// of strip 0) by heavy::root_min (derived A.4).  Not part of the public C-ABI.
#pragma once
#include "amtc_option.cuh"
#include "pwl_device.cuh"
#include "pwl_heavy.cuh"

namespace amtc {

__device__ __forceinline__ Fn root_shfl_fn(const Fn& F, int src) {
    Fn G;
    G.p = reinterpret_cast<const Vtx*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(F.p), src));
    G.n = __shfl_sync(0xffffffffu, F.n, src);
    G.sl = __shfl_sync(0xffffffffu, F.sl, src);
    G.stride = __shfl_sync(0xffffffffu, F.stride, src);
    return G;
}

// mine: this lane's level-1 function (lanes 0, 1 of strip 0 hold (1,0), (1,1));
// writes q->ask (seller) or q->bid (buyer) and the optional root hedge; returns
// the device status bits
static __device__ __noinline__ int tc_root(Fn mine, OptionConsts oc, bool seller, Quote* q, double* hedge,
                                           int lane) {
    const Fn Ur = root_shfl_fn(mine, 0), Dr = root_shfl_fn(mine, 1);
    // quotes at t = 0: S0 both ways, or (1 +- k) S0 with AMTC_COST_AT_T0 (NEXT #3)
    const bool c0 = (oc.flags & FLAG_COST_T0) != 0;
    const double lo = c0 ? -(1.0 + oc.k) * oc.S0 : -oc.S0, hi = c0 ? -(1.0 - oc.k) * oc.S0 : -oc.S0;
    double slW, srW, ymin;
    const double v0 = heavy::root_min(Ur, Dr, lo, hi, slW, srW, ymin, lane);
    // the infimum is finite iff W - hi y decreases on the left and W - lo y increases on the right
    if (!(slW - hi < 0.0) || !(srW - lo > 0.0)) return DEV_UNBOUNDED;
    if (lane == 0) {
        double xi, zeta;
        option_payoff(oc, oc.S0, xi, zeta);
        // u_0(0) of the seller (vertex (zeta, xi)) / buyer (vertex (-zeta, -xi)), slopes lo | hi;
        // a European option cannot be exercised at t = 0
        const double ua = xi + (0.0 < zeta ? lo : hi) * (0.0 - zeta);
        const double ub = -xi + (0.0 < -zeta ? lo : hi) * (0.0 + zeta);
        const bool euro = (oc.flags & FLAG_EUROPEAN) != 0;
        if (seller) q->ask = euro ? v0 : fmax(ua, v0);  // pi^a = z_0(0)
        else q->bid = -(euro ? v0 : fmin(ub, v0));      // pi^b = -z'_0(0)
        if (hedge) *hedge = c0 ? NAN : ymin;            // the position taken at t = 0 (NEXT #2)
    }
    return DEV_OK;
}

}  // namespace amtc
