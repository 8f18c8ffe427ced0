"""Oracle for NEXT row F4: the control plane -- Alg. 1 (adaptive module migration) and
Alg. 2 (load-aware request scheduling), PAPER.md:377-525 (§4.4), written out step by
step in the paper's order with plain Python loops (small inputs only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The product implementation is
paper_2510_13223_b200/csrc/policy.cpp; the two share no code.

Readings (R-F4a..R-F4g) where the pseudo-code is silent or garbled:
  R-F4a  Alg. 2 "Select(candidates, least-loaded)" uses the loads as updated so far;
         ties break by queue length, then instance index.  "lowest-queue" ties break by
         load, then index.
  R-F4b  an assignment enqueues the request: q_len[target] += 1 in both branches.
  R-F4c  load[target] += EstimateLoad(req) only in the least-loaded branch (line 15);
         the lowest-queue branch (lines 17-18) updates no load, as printed.
  R-F4d  Alg. 1 line 11 "load[d_n] - load[d_u]" reads load[d_o] - load[d_u] (A18);
         d_o = most loaded overloaded device, d_u = least loaded underloaded device
         other than d_o (ties: lowest index); the sets are recomputed every iteration.
  R-F4e  a move is executed only if Benefit/Cost >= rho (eq. 35), Benefit =
         Delta_before - Delta_after with Delta_after = |(load_o - u) - (load_u + u)|;
         a layer move that fails the gate falls through to a KV-head move (the finer
         grain); if no move passes, the cycle ends (else Alg. 1 would
         loop forever).
  R-F4f  moving a module moves its load share u and the module itself (counts update).
  R-F4g  hysteresis: a cycle classifies with delta_up when the previous
         cycle migrated nothing, and with delta_down (< delta_up) while migrating.
"""
from __future__ import annotations


def utilization(c: float, c_max: float, m: float, m_max: float) -> float:
    """eq. 32 / eq. 37: U = C / C_max + M / M_max (0 .. 2)."""
    return c / c_max + m / m_max


def dispatch(load, q_len, est_load, delta_l):
    """Alg. 2.  Returns (assignment per request, final load, q_len)."""
    load = [float(x) for x in load]
    q_len = [int(x) for x in q_len]
    n = len(load)
    assign = []
    for r in range(len(est_load)):
        # line 12: least-loaded candidate (R-F4a)
        best = 0
        for i in range(1, n):
            if (load[i], q_len[i], i) < (load[best], q_len[best], best):
                best = i
        if load[best] < delta_l:                      # line 13
            target = best
            load[target] += float(est_load[r])        # line 15 (R-F4c)
        else:                                         # lines 16-18: lowest queue
            target = 0
            for i in range(1, n):
                if (q_len[i], load[i], i) < (q_len[target], load[target], target):
                    target = i
        q_len[target] += 1                            # R-F4b
        assign.append(target)
    return assign, load, q_len


def plan_migrations(load, n_layers, layer_load, layer_cost, n_heads, head_load, head_cost,
                    supports_layer, supports_attn, delta, rho, max_moves=10_000):
    """Alg. 1 for one control cycle.  Returns (moves, final load,
    n_layers, n_heads); a move is (kind, d_o, d_u) with kind 0 = layer, 1 = KV heads."""
    load = [float(x) for x in load]
    n_layers = [int(x) for x in n_layers]
    n_heads = [int(x) for x in n_heads]
    D = len(load)
    moves = []
    while len(moves) < max_moves:
        lo, hi = min(load), max(load)
        overload = [d for d in range(D) if load[d] - lo > delta]          # eq. 33
        underload = [d for d in range(D) if hi - load[d] > delta]
        if not overload or not underload:
            break
        d_o = overload[0]
        for d in overload:
            if load[d] > load[d_o]:
                d_o = d
        cands = [d for d in underload if d != d_o]
        if not cands:
            break
        d_u = cands[0]
        for d in cands:
            if load[d] < load[d_u]:
                d_u = d
        gap = load[d_o] - load[d_u]                                          # eq. 34 (R-F4d)
        done = False
        for kind in (0, 1):                                                  # lines 12-16
            if gap < delta:
                break
            if kind == 0 and not (supports_layer[d_o] and n_layers[d_o] > 0):
                continue
            if kind == 1 and not (supports_attn[d_o] and n_heads[d_o] > 0):
                continue
            u = float(layer_load[d_o] if kind == 0 else head_load[d_o])
            cost = float(layer_cost[d_o] if kind == 0 else head_cost[d_o])
            after = abs((load[d_o] - u) - (load[d_u] + u))
            benefit = gap - after                                            # eq. 35
            if cost > 0 and benefit / cost >= rho:
                load[d_o] -= u                                               # line 17 (R-F4f)
                load[d_u] += u
                if kind == 0:
                    n_layers[d_o] -= 1
                    n_layers[d_u] += 1
                else:
                    n_heads[d_o] -= 1
                    n_heads[d_u] += 1
                moves.append((kind, d_o, d_u))
                done = True
                break
        if not done:
            break
    return moves, load, n_layers, n_heads


def run_cycles(cycles, delta_up, delta_down, rho):
    """Alg. 1 applied once per control period with the hysteresis of PAPER.md:462
    ("distinct upward and downward thresholds (delta_up, delta_down)", reading R-F4g):
    a cycle classifies devices with delta_up while the controller is idle -- the previous
    cycle moved nothing (and before the first cycle) -- and with delta_down while it is
    migrating -- the previous cycle moved at least one module.

    ``cycles``: a list of dicts with the keyword arguments of plan_migrations except
    delta / rho (each period's measured loads and module tables).  Returns the list of
    plan_migrations results, one per cycle."""
    migrating = False
    out = []
    for c in cycles:
        delta = delta_down if migrating else delta_up
        res = plan_migrations(delta=delta, rho=rho, **c)
        migrating = len(res[0]) > 0
        out.append(res)
    return out
