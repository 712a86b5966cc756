// tools/lane_host.cpp -- HOST harness of the product's per-lane node update
// (paper_1110_2477_b200/csrc/pwl_lane.cuh compiled for the CPU).  It runs the
// whole backward induction with lane_node_update on every node, so the
// not-gpu test suite can check the product algebra against the oracle without
// a GPU (tests/test_lane_host.py).  Not part of the product path.
//
// stdin: one option per line "S0 K K2 T sigma R k kind N"
// stdout: "ask bid max_vertices status" per line
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_1110_2477_b200/csrc/pwl_lane.cuh"
using namespace amtc;

static int price_party(double S0, double K, double K2, double T, double sg, double R, double k, int kind, int N,
                       int party, double& price, int& maxn) {
    const double h = sg * std::sqrt(T / N), rho = R * T / N;
    if (!(rho < h && -h < rho)) return 2;
    const bool seller = party == 0;
    auto S_at = [&](int t, int j) { return S0 * std::exp(h * (double)(t - 2 * j)); };
    auto disc = [&](int t) { return std::exp(-rho * (double)t); };
    auto payoff = [&](double S, double& xi, double& zeta) {
        if (kind == 0) { xi = K; zeta = -1.0; }
        else if (kind == 1) { xi = -K; zeta = 1.0; }
        else { xi = std::fmax(S - K, 0.0) - std::fmax(S - K2, 0.0); zeta = 0.0; }
    };
    std::vector<std::vector<Vtx>> z(N + 2);
    std::vector<double> sl(N + 2);
    for (int j = 0; j <= N + 1; ++j) {
        const double Sd = S_at(N + 1, j) * disc(N + 1);
        z[j] = {Vtx{0.0, 0.0, -(1.0 - k) * Sd}};
        sl[j] = -(1.0 + k) * Sd;
    }
    maxn = 1;
    for (int t = N; t >= 0; --t) {
        for (int j = 0; j <= t; ++j) {
            const double S = S_at(t, j), dsc = disc(t);
            const double ka = (t == 0) ? 0.0 : k;  // no costs at t = 0
            const double lo = -(1.0 + ka) * S * dsc, hi = -(1.0 - ka) * S * dsc;
            double xi, zeta;
            payoff(S, xi, zeta);
            const double ux = seller ? zeta : -zeta, uf = (seller ? xi : -xi) * dsc;
            const Fn U = make_fn(z[j].data(), (int)z[j].size(), sl[j]);
            const Fn D = make_fn(z[j + 1].data(), (int)z[j + 1].size(), sl[j + 1]);
            const int cap = 4 * (U.n + D.n) + 16;
            std::vector<Vtx> buf(cap), out(cap);
            Emit E;
            E.out = out.data();
            E.cap = cap;
            E.stride = 1;
            int e = lane_node_update(U, D, lo, hi, ux, uf, seller, buf.data(), cap, 1, E);
            if (e) return e == DEV_UNBOUNDED ? 4 : 3;
            z[j].assign(out.begin(), out.begin() + E.m);
            sl[j] = E.sl;
            if (E.m > maxn) maxn = E.m;
        }
    }
    // z_0 at y = 0
    const Fn Z = make_fn(z[0].data(), (int)z[0].size(), sl[0]);
    int p = -1;
    while (p + 1 < Z.n && Z.v(p + 1).x <= 0.0) ++p;
    const double z0 = piece_at(Z, p, 0.0);
    price = seller ? z0 : -z0;
    return 0;
}

int main() {
    double S0, K, K2, T, sg, R, k;
    int kind, N;
    while (std::scanf("%lf %lf %lf %lf %lf %lf %lf %d %d", &S0, &K, &K2, &T, &sg, &R, &k, &kind, &N) == 9) {
        double ask = NAN, bid = NAN;
        int m0 = 0, m1 = 0;
        int st = price_party(S0, K, K2, T, sg, R, k, kind, N, 0, ask, m0);
        if (!st) st = price_party(S0, K, K2, T, sg, R, k, kind, N, 1, bid, m1);
        std::printf("%.17g %.17g %d %d\n", ask, bid, m0 > m1 ? m0 : m1, st);
    }
    return 0;
}
