"""Host check of the product's per-lane PWL algebra (pwl_lane.cuh compiled for
the CPU by tools/lane_host.cpp) against the oracle: the whole backward
induction, every node updated by lane_node_update, prices compared at the GPU
parity tolerance (tests/tolerance.py, reading A19).  This pins the
device algebra without a GPU; the GPU tests then pin the kernels around it."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from tolerance import close
from paper_1110_2477_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "lane_host.cpp")
BIN = os.path.join(ROOT, "tools", "lane_host")
DEPS = [SRC] + [os.path.join(ROOT, "paper_1110_2477_b200", "csrc", f) for f in ("pwl_lane.cuh", "pwl_device.cuh")]


@pytest.fixture(scope="module")
def lane_host():
    if not os.path.exists(BIN) or any(os.path.getmtime(d) > os.path.getmtime(BIN) for d in DEPS):
        subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", BIN, SRC], check=True)
    return BIN


def run(bin_, batch, N):
    lines = []
    for i in range(len(batch)):
        r = batch.row(i)
        lines.append(f"{r['S0']!r} {r['K']!r} {r['K2']!r} {r['T']!r} {r['sigma']!r} {r['R']!r} {r['k']!r} "
                     f"{r['kind']} {N}")
    out = subprocess.run([bin_], input="\n".join(lines) + "\n", capture_output=True, text=True, check=True).stdout
    return [tuple(float(v) for v in ln.split()) for ln in out.strip().splitlines()]


def check(got, batch, N):
    bad = []
    for i, (ask, bid, maxn, st) in enumerate(got):
        r = batch.row(i)
        q = O.price_tc(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], r["k"], r["kind"], r["K2"]), N)
        assert int(st) == q.status, (i, r, st, q)
        if q.status:
            continue
        if not (close(ask, q.ask, N, r["S0"]) and close(bid, q.bid, N, r["S0"])):
            bad.append((i, r, ask, q.ask, bid, q.bid))
    assert not bad, bad[:3]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 7, 16, 45])
def test_lane_algebra_random(lane_host, N):
    b = W.random_small(60, seed=500 + N, k_max=0.05)
    check(run(lane_host, b, N), b, N)


def test_lane_algebra_large_k(lane_host):
    """k up to 30%: many breakpoints, buyer non-convexity everywhere."""
    b = W.random_small(40, seed=77, k_max=0.3)
    check(run(lane_host, b, 30), b, 30)


def test_lane_algebra_k0_is_crr(lane_host):
    b = W.random_small(30, seed=9, k_max=0.0)
    got = run(lane_host, b, 50)
    for i, (ask, bid, _, st) in enumerate(got):
        r = b.row(i)
        crr = O.price_crr(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], 0.0, r["kind"], r["K2"]), 50)
        assert st == 0
        assert abs(ask - crr) <= 1e-9 * crr + 1e-10 and abs(bid - crr) <= 1e-9 * crr + 1e-10


def test_lane_algebra_config4_sample(lane_host):
    """A few BASELINE config-4 options at N = 300 (heavy buyer sawtooth for calls)."""
    b = W.config4()
    idx = np.random.default_rng(3).choice(len(b), 12, replace=False)
    sub = b.subset(idx)
    check(run(lane_host, sub, 300), sub, 300)
