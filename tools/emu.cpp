// tools/emu.cpp -- DEVELOPER TOOL: runs the device node-update algebra
// (paper_1110_2477_b200/csrc/pwl_device.cuh) sequentially on the host to debug
// representation sizes.  Not part of the product path, not used by tests.
#include <math.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1110_2477_b200/csrc/pwl_device.cuh"
using namespace amtc;

int main(int argc, char** argv) {
    if (argc < 10) { fprintf(stderr, "usage: emu S0 K K2 T sigma R k kind N [party]\n"); return 2; }
    double S0 = atof(argv[1]), K = atof(argv[2]), K2 = atof(argv[3]), T = atof(argv[4]), sg = atof(argv[5]),
           R = atof(argv[6]), k = atof(argv[7]);
    int kind = atoi(argv[8]), N = atoi(argv[9]);
    int p0 = argc > 10 ? atoi(argv[10]) : 0, p1 = argc > 10 ? atoi(argv[10]) : 1;
    double h = sg * sqrt(T / N), rho = R * T / N;
    for (int party = p0; party <= p1; ++party) {
        std::vector<std::vector<Vtx>> z(N + 2);
        std::vector<double> sl(N + 2);
        for (int j = 0; j <= N + 1; ++j) {
            double Sd = S0 * exp(h * (N + 1 - 2 * j)) * exp(-rho * (N + 1));
            z[j] = {Vtx{0.0, 0.0, -(1 - k) * Sd}};
            sl[j] = -(1 + k) * Sd;
        }
        long long vsum = 0;
        int excess = -1000, small_in_large_out_min = 1000;
        int maxn = 0;
        for (int t = N; t >= 1; --t) {
            double disc = exp(-rho * t);
            int lvmax = 0;
            for (int j = 0; j <= t; ++j) {
                double S = S0 * exp(h * (t - 2 * j));
                double lo = -(1 + k) * S * disc, hi = -(1 - k) * S * disc;
                double xi, zeta;
                if (kind == 0) { xi = K; zeta = -1; } else if (kind == 1) { xi = -K; zeta = 1; }
                else { xi = fmax(S - K, 0.0) - fmax(S - K2, 0.0); zeta = 0; }
                const Fn U = make_fn(z[j].data(), (int)z[j].size(), sl[j]);
                const Fn D = make_fn(z[j + 1].data(), (int)z[j + 1].size(), sl[j + 1]);
                int b = 4 * (U.n + D.n) + 16;
                std::vector<Vtx> r0(b), r1(b);
                int nZ; double slZ;
                int err = node_update(U, D, lo, hi, party == 0 ? zeta : -zeta, (party == 0 ? xi : -xi) * disc,
                                      party == 0, r0.data(), r1.data(), b, nZ, slZ);
                if (err) { printf("err %d at t=%d j=%d\n", err, t, j); return 1; }
                if (nZ - (U.n + D.n) > excess) excess = nZ - (U.n + D.n);
                if (U.n + D.n <= 8 && nZ > 4 && (U.n + D.n) < small_in_large_out_min) small_in_large_out_min = U.n + D.n;
                z[j].assign(r1.begin(), r1.begin() + nZ);
                sl[j] = slZ;
                vsum += nZ;
                if (nZ > lvmax) lvmax = nZ;
            }
            if (lvmax > maxn) maxn = lvmax;
            if (getenv("EMU_DUMP") && lvmax >= atoi(getenv("EMU_DUMP"))) {
                for (int j = 0; j <= t; ++j) if ((int)z[j].size() == lvmax) {
                    printf("dump t=%d j=%d n=%d sl=%.17g\n", t, j, lvmax, sl[j]);
                    for (auto& v : z[j]) printf("  x=%.17g f=%.17g s=%.17g\n", v.x, v.f, v.s);
                    break;
                }
                return 0;
            }
            if (getenv("EMU_TRACE") && (t % (N / 10 > 0 ? N / 10 : 1) == 0)) printf("  t=%d level max=%d\n", t, lvmax);
        }
        // root
        std::vector<Vtx> w(4 * (z[0].size() + z[1].size()) + 16);
        const Fn U = make_fn(z[0].data(), (int)z[0].size(), sl[0]);
        const Fn D = make_fn(z[1].data(), (int)z[1].size(), sl[1]);
        Emit E; E.out = w.data(); E.cap = (int)w.size();
        envelope(U, D, true, E);
        double mv = INFINITY;
        for (int i = 0; i < E.m; ++i) mv = fmin(mv, fma(S0, w[i].x, w[i].f));
        double xi, zeta;
        if (kind == 0) { xi = K; zeta = -1; } else if (kind == 1) { xi = -K; zeta = 1; }
        else { xi = fmax(S0 - K, 0.0) - fmax(S0 - K2, 0.0); zeta = 0; }
        double intr = xi + zeta * S0;
        double price = party == 0 ? fmax(intr, mv) : fmax(intr, -mv);
        printf("party=%d price=%.15g maxn=%d avgn=%.3f excess(nZ-nU-nD)=%d\n", party, price, maxn, (double)vsum / ((N + 1.0) * N / 2), excess);
    }
    return 0;
}
