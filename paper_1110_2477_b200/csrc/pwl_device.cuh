// pwl_device.cuh -- device-side piecewise-linear (PWL) algebra for the
// Roux-Zastawniak seller/buyer node recursion (Sec. 3).
//
// Representation (product path; independent of the CPU oracle): a continuous
// PWL function of the share holding y is a sorted vertex list
//     v[i] = (x_i, f_i, s_i),  i = 0..n-1,  n >= 1,
// where f_i = f(x_i) and s_i is the slope on (x_i, x_{i+1}) (s_{n-1} is the
// right tail), plus the left-tail slope sl on (-inf, x_0).  A line is a single
// anchor vertex with s_0 == sl.  Slopes are carried EXACTLY: every slope is a
// copy of a lattice value -(1 +- k) S_{t,j} r^-t created once (as a quote or a
// tail) and never recomputed, so "same slope" is a bitwise test and no
// difference quotient is ever taken.
//
// All functions are stored DISCOUNTED to time 0: zh_t = z_t / r^t.  Then the
// paper's "w_t / r" disappears: wh_t = max(zh_{t+1}^u, zh_{t+1}^d)
// = (w_t / r) / r^t, and the slope restriction to [-S^a_t, -S^b_t] becomes a
// restriction to [-S^a_t r^-t, -S^b_t r^-t] (restriction commutes with
// positive scaling).  At t = 0, r^0 = 1, so prices read off unchanged.
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define AMTC_HD __host__ __device__ __forceinline__
#else
#define AMTC_HD inline
#endif

namespace amtc {

struct Vtx {
    double x, f, s;
};

// status bits raised by the device algebra
enum : int { DEV_OK = 0, DEV_OVERFLOW = 1, DEV_UNBOUNDED = 2 };

// Rounding guards (reading R10: they change values by rounding-level amounts
// only and keep the representation free of rounding-made micro-pieces):
//  * two values closer than TOL_F (|a| + |b| + 1) are "equal": a function does
//    not "cross" another it merely touches (ties are broken by slope);
//  * a piece shorter than TOL_X (1 + |x|) is folded into its neighbour.
constexpr double TOL_F = 1e-14;
#ifndef AMTC_TOL_X
#define AMTC_TOL_X 1e-13
#endif
constexpr double TOL_X = AMTC_TOL_X;
AMTC_HD double ftol(double a, double b) { return TOL_F * (fabs(a) + fabs(b) + 1.0); }
AMTC_HD double xtol(double x) { return TOL_X * (1.0 + fabs(x)); }

// Forward emitter: appends vertices in increasing x, skipping non-kinks
// (same slope as the previous piece) and folding zero-length pieces.
// STR > 0: compile-time element stride of `out` (shared-memory rows of the
// light kernel); STR = 0: the runtime `stride` member.
template <int STR = 0>
struct EmitT {
    Vtx* out;
    int m, cap;
    int stride;     // element stride of `out` when STR == 0 (1 = contiguous; 32 = lane-interleaved slots)
    double sl;      // left-tail slope of the function being built
    double last_s;  // slope of the last piece emitted (sl if none)
    double ax, af;  // anchor candidate (first point offered)
    bool has_anchor;
    int err;

    AMTC_HD void init(Vtx* o, int c, double left_slope, int str = 1) {
        out = o; m = 0; cap = c; stride = str; sl = left_slope; last_s = left_slope; has_anchor = false;
        err = DEV_OK;
    }
    AMTC_HD Vtx& at(int i) { return out[i * (STR ? STR : stride)]; }
    AMTC_HD void push(double x, double f, double s) {
        if (!has_anchor) { ax = x; af = f; has_anchor = true; }
        if (s == last_s) return;  // not a kink
        if (m > 0 && !(x > at(m - 1).x + xtol(x))) {
            // (near) zero-length piece (coincident or rounding-made vertex):
            // the previous vertex turns directly into slope s
            at(m - 1).s = s;
            double left = (m > 1) ? at(m - 2).s : sl;
            if (left == s) m--;  // the previous vertex is no longer a kink
            last_s = s;
            return;
        }
        if (m >= cap) { err |= DEV_OVERFLOW; return; }
        Vtx& o = at(m);
        o.x = x; o.f = f; o.s = s;
        m++;
        last_s = s;
    }
    // close the function: a line keeps one anchor vertex
    AMTC_HD int finish() {
        if (m == 0) {
            if (cap < 1) { err |= DEV_OVERFLOW; return 0; }
            at(0).x = has_anchor ? ax : 0.0;
            at(0).f = has_anchor ? af : 0.0;
            at(0).s = sl;
            m = 1;
        }
        return m;
    }
};
using Emit = EmitT<0>;

// A read-only function view (STR > 0: compile-time element stride).
template <int STR = 0>
struct FnT {
    const Vtx* p;
    int n;
    double sl;
    int stride;  // element stride of p when STR == 0 (1 = contiguous; 32 = lane-interleaved slots)
    AMTC_HD const Vtx& v(int i) const { return p[i * (STR ? STR : stride)]; }
    AMTC_HD double slope_right(int i) const { return i < 0 ? sl : v(i).s; }
};
using Fn = FnT<0>;
AMTC_HD Fn make_fn(const Vtx* p, int n, double sl, int stride = 1) {
    Fn F;
    F.p = p; F.n = n; F.sl = sl; F.stride = stride;
    return F;
}
template <int STR>
AMTC_HD FnT<STR> make_fn_s(const Vtx* p, int n, double sl) {
    FnT<STR> F;
    F.p = p; F.n = n; F.sl = sl; F.stride = STR;
    return F;
}

// value at y of the piece that starts at vertex i (i = -1: the left tail,
// anchored at vertex 0)
template <int STR>
AMTC_HD double piece_at(const FnT<STR>& F, int i, double y) {
    const Vtx& a = F.v(i < 0 ? 0 : i);
    double s = i < 0 ? F.sl : a.s;
    return fma(s, y - a.x, a.f);
}

}  // namespace amtc
