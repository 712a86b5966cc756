"""Brute-force definitions of the ask and bid prices on tiny trees (test-only).

This module shares nothing with the oracle: it never builds a PWL function and
never runs the recursion.  It writes the superhedging problem of P:92 ("the
minimum amount of wealth that the seller ... needs to hedge his/her positions in
all circumstances"; "the maximum amount of wealth that the buyer can borrow
against the right to exercise") as linear programs over the NON-recombining
path tree, with the market of Sec. 3/4.1:

  * levels t = 0..N+1 (the extra instant N+1 with payoff (0,0));
  * stock S = S0 u^(#up - #down); quotes Sa = (1+k)S, Sb = (1-k)S for t >= 1
    and Sa = Sb = S0 at t = 0;
  * cash grows by r per step.

Variables at every path node nu: the holding (X, Y) entering nu and, for
t <= N, the post-trade holding (P, Q).  Self-financing trade at the quotes:
    P + Sa (Q - Y) <= X   and   P + Sb (Q - Y) <= X
(the two constraints together are exactly "buy at ask, sell at bid").
Children mu of nu: X_mu = r P_nu, Y_mu = Q_nu.  Root: Y = 0.

Seller (ask): cover the exercise obligation (xi, zeta) at EVERY node (the holder
may exercise at any t <= N; at N+1 the obligation is (0,0)):
    X + Sb (Y - zeta) >= xi   and   X + Sa (Y - zeta) >= xi .
ask = min X_root.

Buyer (bid): for a stopping time tau (a set of stop nodes, one per path, with a
forced stop at N+1), cover -(xi, zeta) at the stop nodes only:
    X + Sb (Y + zeta) >= -xi  and  X + Sa (Y + zeta) >= -xi ,
no trading constraints after tau.  bid = max over tau of (-min X_root).
Stopping times are enumerated exhaustively (5, 26, 677 of them for N = 1, 2, 3).
"""
from __future__ import annotations

import itertools
import math

import numpy as np
from scipy.optimize import linprog

PUT, CALL, BULL = 0, 1, 2


def _payoff(kind, K, K2, S):
    if kind == PUT:
        return K, -1.0
    if kind == CALL:
        return -K, 1.0
    return max(S - K, 0.0) - max(S - K2, 0.0), 0.0


def _tree(S0, T, sigma, R, k, N, cost_t0=False):
    u = math.exp(sigma * math.sqrt(T / N))
    d = 1.0 / u
    r = math.exp(R * T / N)
    nodes = []  # (t, m=#up-#down, parent index, path)
    index = {}
    for t in range(N + 2):
        for path in itertools.product((0, 1), repeat=t):  # 0 = up, 1 = down
            m = sum(1 if b == 0 else -1 for b in path)
            parent = index[path[:-1]] if t > 0 else -1
            index[path] = len(nodes)
            nodes.append((t, m, parent, path))
    quotes = []
    for (t, m, _, _) in nodes:
        S = S0 * u ** m
        if t == 0 and not cost_t0:  # no costs at t = 0 unless the variant asks for them
            quotes.append((S, S0, S0))
        else:
            quotes.append((S, (1 + k) * S, (1 - k) * S))
    return nodes, quotes, r


def _solve(nodes, quotes, r, N, cover_rows):
    """min X_root subject to trading before stop nodes and cover at stop nodes.
    cover_rows: dict node -> (xi', zeta') meaning X >= u(Y) with u built from
    (xi', zeta') as in Eq. (1):  X + Sb (Y - zeta') >= xi', X + Sa (Y - zeta') >= xi'.
    Nodes below a stop node are dropped."""
    active = []
    stopped_anc = set()
    for i, (t, m, parent, path) in enumerate(nodes):
        if parent >= 0 and (parent in stopped_anc or parent in cover_rows):
            stopped_anc.add(i)
            continue
        active.append(i)
    pos = {}
    nv = 0
    for i in active:
        t = nodes[i][0]
        trade = (i not in cover_rows) and t <= N
        pos[i] = (nv, nv + 1, nv + 2 if trade else -1, nv + 3 if trade else -1)
        nv += 4 if trade else 2
    A_ub, b_ub, A_eq, b_eq = [], [], [], []
    for i in active:
        t, m, parent, path = nodes[i]
        S, Sa, Sb = quotes[i]
        X, Y, P, Q = pos[i]
        if P >= 0:
            for s in (Sa, Sb):  # P + s (Q - Y) <= X
                row = np.zeros(nv)
                row[P] += 1.0
                row[Q] += s
                row[Y] -= s
                row[X] -= 1.0
                A_ub.append(row)
                b_ub.append(0.0)
        if i in cover_rows:
            xi, zeta = cover_rows[i]
            for s in (Sa, Sb):  # -(X + s (Y - zeta)) <= -xi
                row = np.zeros(nv)
                row[X] -= 1.0
                row[Y] -= s
                A_ub.append(row)
                b_ub.append(-xi - s * zeta)
        if parent >= 0:
            Xp, Yp, Pp, Qp = pos[parent]
            row = np.zeros(nv)
            row[X] = 1.0
            row[Pp] = -r
            A_eq.append(row)
            b_eq.append(0.0)
            row = np.zeros(nv)
            row[Y] = 1.0
            row[Qp] = -1.0
            A_eq.append(row)
            b_eq.append(0.0)
    root = pos[0]
    row = np.zeros(nv)
    row[root[1]] = 1.0
    A_eq.append(row)
    b_eq.append(0.0)
    c = np.zeros(nv)
    c[root[0]] = 1.0
    res = linprog(c, A_ub=np.array(A_ub), b_ub=np.array(b_ub), A_eq=np.array(A_eq), b_eq=np.array(b_eq),
                  bounds=[(None, None)] * nv, method="highs",
                  options={"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise RuntimeError(res.message)
    return res.fun


def ask_lp(S0, K, T, sigma, R, k, N, kind=PUT, K2=0.0, cost_t0=False):
    nodes, quotes, r = _tree(S0, T, sigma, R, k, N, cost_t0)
    cover = {}
    for i, (t, m, parent, path) in enumerate(nodes):
        cover[i] = (0.0, 0.0) if t == N + 1 else _payoff(kind, K, K2, quotes[i][0])
    # the seller covers at every node AND trades at every node t <= N:
    return _solve_seller(nodes, quotes, r, N, cover)


def _solve_seller(nodes, quotes, r, N, cover):
    """Seller: cover at every node and trade at every t <= N (no stopping)."""
    nv = 0
    pos = {}
    for i, (t, m, parent, path) in enumerate(nodes):
        trade = t <= N
        pos[i] = (nv, nv + 1, nv + 2 if trade else -1, nv + 3 if trade else -1)
        nv += 4 if trade else 2
    A_ub, b_ub, A_eq, b_eq = [], [], [], []
    for i, (t, m, parent, path) in enumerate(nodes):
        S, Sa, Sb = quotes[i]
        X, Y, P, Q = pos[i]
        if P >= 0:
            for s in (Sa, Sb):
                row = np.zeros(nv)
                row[P] += 1.0
                row[Q] += s
                row[Y] -= s
                row[X] -= 1.0
                A_ub.append(row)
                b_ub.append(0.0)
        xi, zeta = cover[i]
        for s in (Sa, Sb):
            row = np.zeros(nv)
            row[X] -= 1.0
            row[Y] -= s
            A_ub.append(row)
            b_ub.append(-xi - s * zeta)
        if parent >= 0:
            Xp, Yp, Pp, Qp = pos[parent]
            row = np.zeros(nv)
            row[X] = 1.0
            row[Pp] = -r
            A_eq.append(row)
            b_eq.append(0.0)
            row = np.zeros(nv)
            row[Y] = 1.0
            row[Qp] = -1.0
            A_eq.append(row)
            b_eq.append(0.0)
    row = np.zeros(nv)
    row[pos[0][1]] = 1.0
    A_eq.append(row)
    b_eq.append(0.0)
    c = np.zeros(nv)
    c[pos[0][0]] = 1.0
    res = linprog(c, A_ub=np.array(A_ub), b_ub=np.array(b_ub), A_eq=np.array(A_eq), b_eq=np.array(b_eq),
                  bounds=[(None, None)] * nv, method="highs",
                  options={"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise RuntimeError(res.message)
    return res.fun


def _stopping_times(nodes, N):
    """All stopping times as sets of stop-node indices (forced stop at N+1)."""
    children = {i: [] for i in range(len(nodes))}
    for i, (t, m, parent, path) in enumerate(nodes):
        if parent >= 0:
            children[parent].append(i)

    def rec(i):
        t = nodes[i][0]
        if t == N + 1:
            yield (i,)
            return
        yield (i,)  # stop here
        c0, c1 = children[i]
        for a in rec(c0):
            for b in rec(c1):
                yield a + b

    return list(rec(0))


def bid_enum(S0, K, T, sigma, R, k, N, kind=PUT, K2=0.0, cost_t0=False):
    nodes, quotes, r = _tree(S0, T, sigma, R, k, N, cost_t0)
    best = -math.inf
    for tau in _stopping_times(nodes, N):
        cover = {}
        for i in tau:
            t = nodes[i][0]
            xi, zeta = (0.0, 0.0) if t == N + 1 else _payoff(kind, K, K2, quotes[i][0])
            cover[i] = (-xi, -zeta)  # buyer receives (xi, zeta): Eq. (6) is Eq. (1) with -(xi, zeta)
        best = max(best, -_solve(nodes, quotes, r, N, cover))
    return best


def bid_milp(S0, K, T, sigma, R, k, N, kind=PUT, K2=0.0, cost_t0=False, big_m=1e5):
    """The bid as ONE mixed-integer program: the max over stopping times
    tau of the buyer's LP, with tau encoded by binaries instead of enumerated
    (N = 4 has 458,330 stopping times).  Per path node nu: stop_nu in {0,1},
    alive_nu = 1 - sum of stop over the strict ancestors (alive_root = 1),
    stop_nu <= alive_nu, stop forced (= alive) at t = N+1.  The cover rows of a
    stop node hold exactly when stop_nu = 1 (big-M relaxation otherwise); the
    trading rows are kept at every node (after tau the holdings are unconstrained
    by anything else, so they never bind).  bid = max -X_root."""
    from scipy.optimize import LinearConstraint, milp
    nodes, quotes, r = _tree(S0, T, sigma, R, k, N, cost_t0)
    nn = len(nodes)
    # variables: X, Y, P, Q per node (P, Q unused at t = N+1), then stop per node
    X = lambda i: 4 * i
    Y = lambda i: 4 * i + 1
    P = lambda i: 4 * i + 2
    Q = lambda i: 4 * i + 3
    Z = lambda i: 4 * nn + i
    nv = 5 * nn
    rows, lo, hi = [], [], []

    def add(coefs, l, h):
        row = np.zeros(nv)
        for j, c in coefs:
            row[j] += c
        rows.append(row)
        lo.append(l)
        hi.append(h)

    anc = {}
    for i, (t, m, parent, path) in enumerate(nodes):
        anc[i] = [] if parent < 0 else anc[parent] + [parent]
    for i, (t, m, parent, path) in enumerate(nodes):
        S, Sa, Sb = quotes[i]
        if t <= N:
            for s in (Sa, Sb):  # P + s (Q - Y) <= X
                add([(P(i), 1.0), (Q(i), s), (Y(i), -s), (X(i), -1.0)], -np.inf, 0.0)
        xi, zeta = (0.0, 0.0) if t == N + 1 else _payoff(kind, K, K2, S)
        for s in (Sa, Sb):  # stop_i = 1  =>  X + s (Y + zeta) >= -xi
            add([(X(i), 1.0), (Y(i), s), (Z(i), -big_m)], -xi - s * zeta - big_m, np.inf)
        # stop_i <= alive_i = 1 - sum_{a in anc} stop_a ; '=' at t = N+1
        coefs = [(Z(i), 1.0)] + [(Z(a), 1.0) for a in anc[i]]
        add(coefs, 1.0 if t == N + 1 else 0.0, 1.0)
        if parent >= 0:
            add([(X(i), 1.0), (P(parent), -r)], 0.0, 0.0)
            add([(Y(i), 1.0), (Q(parent), -1.0)], 0.0, 0.0)
    add([(Y(0), 1.0)], 0.0, 0.0)
    c = np.zeros(nv)
    c[X(0)] = 1.0
    lb = np.full(nv, -big_m / 10)
    ub = np.full(nv, big_m / 10)
    lb[4 * nn:] = 0.0
    ub[4 * nn:] = 1.0
    integrality = np.zeros(nv)
    integrality[4 * nn:] = 1
    from scipy.optimize import Bounds
    res = milp(c, constraints=LinearConstraint(np.array(rows), np.array(lo), np.array(hi)),
               integrality=integrality, bounds=Bounds(lb, ub),
               options={"mip_rel_gap": 0.0, "presolve": True})
    if res.status != 0:
        raise RuntimeError(res.message)
    return -res.fun
