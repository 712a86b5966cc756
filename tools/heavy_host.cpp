// tools/heavy_host.cpp -- HOST check of the warp-cooperative node update
// (pwl_heavy.cuh) against the per-lane node update (pwl_lane.cuh) on every node
// of real trees.  Test infrastructure only (tests/test_heavy_host.py).
// stdin: "S0 K K2 T sigma R k kind N" per line; stdout per line:
//   "<nodes> <max vertex excess> <max rel value diff> <status>"
#include "warp_emu.h"
#include <atomic>
// sweep-C piece statistics (0 empty lane, 1 fast piece, 2 general piece, 3 all-fast block)
static std::atomic<long> g_stat[4];
static bool g_count = false;
#define AMTC_HEAVY_STAT(i) (g_count ? (void)g_stat[(i)].fetch_add(1, std::memory_order_relaxed) : (void)0)
#define AMTC_HEAVY_STAT_BLOCKS 1
static std::atomic<long> g_why[32];
#define AMTC_WHY(i) (g_count ? (void)g_why[(i)].fetch_add(1) : (void)0)
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <string>
#include "../paper_1110_2477_b200/csrc/pwl_lane.cuh"
#include "../paper_1110_2477_b200/csrc/pwl_heavy.cuh"
using namespace amtc;

static double eval(const std::vector<Vtx>& z, double sl, double y) {
    const Fn F = make_fn(z.data(), (int)z.size(), sl);
    int p = -1;
    while (p + 1 < F.n && F.v(p + 1).x <= y) ++p;
    return piece_at(F, p, y);
}

int main(int argc, char** argv) {
    // argv: [tl [v [stop]]]: nodes with more than tl child vertices take the
    // warp path and its result feeds the next level (as on the GPU); tl < 0:
    // every node is checked but the lane result is kept
    const int tl = argc > 1 ? std::atoi(argv[1]) : -1;
    const int verbose = argc > 2;
    // HEAVY_VARIANT=lane: the lane-contiguous update; default: the block-synchronous one
    const char* hv = std::getenv("HEAVY_VARIANT");
    const bool block_variant = !(hv && std::string(hv) == "lane");
    double S0, K, K2, T, sg, R, k;
    int kind, N;
    while (std::scanf("%lf %lf %lf %lf %lf %lf %lf %d %d", &S0, &K, &K2, &T, &sg, &R, &k, &kind, &N) == 9) {
        const double h = sg * std::sqrt(T / N), rho = R * T / N;
        long nodes = 0;
        int worst_excess = -1000000;
        double worst_rel = 0.0;
        int status = 0;
        for (int party = 0; party < 2 && !status; ++party) {
            const bool seller = party == 0;
            auto S_at = [&](int t, int j) { return S0 * std::exp(h * (double)(t - 2 * j)); };
            auto disc = [&](int t) { return std::exp(-rho * (double)t); };
            std::vector<std::vector<Vtx>> z(N + 2);
            std::vector<double> sl(N + 2);
            for (int j = 0; j <= N + 1; ++j) {
                const double Sd = S_at(N + 1, j) * disc(N + 1);
                z[j] = {Vtx{0.0, 0.0, -(1.0 - k) * Sd}};
                sl[j] = -(1.0 + k) * Sd;
            }
            for (int t = N; t >= 1 && !status; --t) {
                for (int j = 0; j <= t && !status; ++j) {
                    const double S = S_at(t, j), dsc = disc(t);
                    const double lo = -(1.0 + k) * S * dsc, hi = -(1.0 - k) * S * dsc;
                    double xi, zeta;
                    if (kind == 0) { xi = K; zeta = -1.0; }
                    else if (kind == 1) { xi = -K; zeta = 1.0; }
                    else { xi = std::fmax(S - K, 0.0) - std::fmax(S - K2, 0.0); zeta = 0.0; }
                    const double ux = seller ? zeta : -zeta, uf = (seller ? xi : -xi) * dsc;
                    const Fn U = make_fn(z[j].data(), (int)z[j].size(), sl[j]);
                    const Fn D = make_fn(z[j + 1].data(), (int)z[j + 1].size(), sl[j + 1]);
                    const int cap = 4 * (U.n + D.n) + 16;
                    std::vector<Vtx> buf(cap), out(cap);
                    Emit E;
                    E.out = out.data(); E.cap = cap; E.stride = 1;
                    if (lane_node_update(U, D, lo, hi, ux, uf, seller, buf.data(), cap, 1, E)) { status = 1; break; }
                    std::vector<Vtx> zl(out.begin(), out.begin() + E.m);
                    // the warp path on the same children
                    std::vector<Vtx> scratch(heavy::scratch_vertices(U.n + D.n) + 4 * (U.n + D.n) + 64),
                        arena(8 * (U.n + D.n) + 64);
                    int counter = 0, zoff = 0, nZ = 0, err = 0;
                    heavy::HWin win;
                    g_count = U.n + D.n > (tl > 0 ? tl : 64);
                    warp_emu::run_warp([&](int lane) {
                        int zo, zn;
                        const int e = block_variant
                            ? (zo = 0, heavy::node_update_block(U, D, lo, hi, ux, uf, seller, &win, scratch.data(),
                                                                (int)scratch.size(), arena.data(), (int)arena.size(),
                                                                zn, lane))
                            : heavy::node_update(U, D, lo, hi, ux, uf, seller, scratch.data(), (int)scratch.size(),
                                                 arena.data(), &counter, (int)arena.size(), zo, zn, lane);
                        if (lane == 0) { err = e; zoff = zo; nZ = zn; }
                    });
                    if (err) { status = 2; if (verbose) std::printf("heavy err %d at t=%d j=%d\n", err, t, j); break; }
                    std::vector<Vtx> zh(arena.begin() + zoff, arena.begin() + zoff + nZ);
                    ++nodes;
                    worst_excess = std::max(worst_excess, (int)zh.size() - (int)zl.size());
                    // compare values at the vertices of both and at +-1 beyond
                    double scale = 1.0;
                    for (auto& v : zl) scale = std::max(scale, std::fabs(v.f));
                    std::vector<double> ys;
                    for (auto& v : zl) ys.push_back(v.x);
                    for (auto& v : zh) ys.push_back(v.x);
                    ys.push_back(zl.front().x - 1.0); ys.push_back(zl.back().x + 1.0);
                    double rel = 0.0;
                    for (double y : ys) rel = std::max(rel, std::fabs(eval(zl, E.sl, y) - eval(zh, lo, y)) / scale);
                    worst_rel = std::max(worst_rel, rel);
                    if (verbose && ((int)zh.size() > (int)zl.size() + 1 || rel > 1e-9)) {
                        std::printf("t=%d j=%d party=%d nU=%d nD=%d lane=%zu heavy=%zu rel=%.3g\n", t, j, party, U.n, D.n,
                                    zl.size(), zh.size(), rel);
                        for (auto& v : zl) std::printf("   L %.17g %.17g %.17g\n", v.x, v.f, v.s);
                        for (auto& v : zh) std::printf("   H %.17g %.17g %.17g\n", v.x, v.f, v.s);
                        if (argc > 3) return 0;
                    }
                    const bool use_heavy = tl >= 0 && U.n + D.n > tl;
                    z[j] = use_heavy ? zh : zl;
                    sl[j] = use_heavy ? lo : E.sl;
                }
            }
        }
        std::printf("%ld %d %.3g %d\n", nodes, worst_excess, worst_rel, status);
        std::fprintf(stderr, "pieces: fast %ld general %ld empty-lane %ld all-fast blocks %ld\n", g_stat[1].load(),
                     g_stat[2].load(), g_stat[0].load(), g_stat[3].load());
        for (int i = 0; i < 32; ++i) if (g_why[i]) std::fprintf(stderr, " why %d: %ld\n", i, g_why[i].load());
        std::fflush(stdout);
    }
    return 0;
}
