"""Host check of the warp-cooperative (heavy) node update, pwl_heavy.cuh,
against the per-lane node update, pwl_lane.cuh (itself pinned to the oracle by
test_lane_host.py).  tools/heavy_host.cpp runs the device header on the CPU
with the warp collectives emulated by 32 threads (tools/warp_emu.h), on every
node of real trees; a small heavy threshold also feeds the warp path's results
forward, as the GPU does.  Checks: equal values (relative 1e-11 of the node's
scale) and no representation bloat (at most one extra vertex per node)."""
import os
import subprocess

import pytest

from paper_1110_2477_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "heavy_host.cpp")
BIN = os.path.join(ROOT, "tools", "heavy_host")
DEPS = [SRC, os.path.join(ROOT, "tools", "warp_emu.h")] + [
    os.path.join(ROOT, "paper_1110_2477_b200", "csrc", f) for f in ("pwl_lane.cuh", "pwl_device.cuh", "pwl_heavy.cuh")]


@pytest.fixture(scope="module")
def heavy_host():
    if not os.path.exists(BIN) or any(os.path.getmtime(d) > os.path.getmtime(BIN) for d in DEPS):
        subprocess.run(["g++", "-O2", "-std=c++20", "-pthread", "-o", BIN, SRC], check=True)
    return BIN


def run(bin_, lines, tl):
    out = subprocess.run([bin_, str(tl)], input="\n".join(lines) + "\n", capture_output=True, text=True,
                         check=True, timeout=600).stdout
    return [ln.split() for ln in out.strip().splitlines()]


def option_lines(batch, N):
    return [f"{r['S0']!r} {r['K']!r} {r['K2']!r} {r['T']!r} {r['sigma']!r} {r['R']!r} {r['k']!r} {r['kind']} {N}"
            for r in (batch.row(i) for i in range(len(batch)))]


@pytest.mark.parametrize("tl", [2, 6])
def test_heavy_matches_lane_forced(heavy_host, tl):
    b = W.random_small(6, seed=700 + tl, k_max=0.08)
    for nodes, excess, rel, st in run(heavy_host, option_lines(b, 18), tl):
        assert st == "0"
        assert int(excess) <= 1
        assert float(rel) < 1e-11


def test_heavy_matches_lane_sawtooth(heavy_host):
    """A call at large k/h (the buyer's sawtooth grows to ~40 vertices at N = 80).
    Nodes above 16 child vertices feed the warp path's result forward; both
    branches of sweep C (the z = W fast path and the general emission) must
    occur on the sawtooth (the harness counts them on stderr)."""
    line = "100.0 106.5 0.0 0.6 0.3 0.018 0.017 1 80"
    p = subprocess.run([heavy_host, "16"], input=line + "\n", capture_output=True, text=True, check=True, timeout=600)
    for nodes, excess, rel, st in (ln.split() for ln in p.stdout.strip().splitlines()):
        assert st == "0" and int(excess) <= 1 and float(rel) < 1e-11
    stats = p.stderr.split()
    fast, general = int(stats[stats.index("fast") + 1]), int(stats[stats.index("general") + 1])
    assert fast > 0 and general > 0
