"""NEXT row F4: control plane over the migration mechanisms (§4.4).

Thin binding over the C++ policy in ``csrc/policy.cpp`` (``bs_dispatch_requests`` =
Alg. 2, ``bs_plan_migrations`` = one cycle of Alg. 1) plus the stateful hysteresis of
PAPER.md:462 (reading R-F4g): a cycle classifies devices with ``delta_up`` while the
controller is idle and with ``delta_down`` once it has started migrating.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _check, lib


def utilization(c: float, c_max: float, m: float, m_max: float) -> float:
    """eq. 32 / eq. 37."""
    return lib().bs_utilization(c, c_max, m, m_max)


def _arr(x, dtype):
    return np.ascontiguousarray(np.asarray(x, dtype=dtype))


def dispatch(load, q_len, est_load, delta_l: float):
    """Alg. 2: returns (assignment list, final load, final q_len)."""
    ld = _arr(load, np.float64).copy()
    ql = _arr(q_len, np.int32).copy()
    est = _arr(est_load, np.float64)
    out = np.zeros(max(len(est), 1), dtype=np.int32)
    _check(lib().bs_dispatch_requests(len(ld), ld.ctypes.data, ql.ctypes.data, len(est),
                                      est.ctypes.data if len(est) else None, float(delta_l),
                                      out.ctypes.data))
    return out[:len(est)].tolist(), ld.tolist(), ql.tolist()


def plan_migrations(load, n_layers, layer_load, layer_cost, n_heads, head_load, head_cost,
                    supports_layer, supports_attn, delta: float, rho: float, max_moves: int = 10_000):
    """One cycle of Alg. 1: returns (moves [(kind, from, to)], load, n_layers, n_heads)."""
    ld = _arr(load, np.float64).copy()
    nl = _arr(n_layers, np.int32).copy()
    nh = _arr(n_heads, np.int32).copy()
    ll, lc = _arr(layer_load, np.float64), _arr(layer_cost, np.float64)
    hl, hc = _arr(head_load, np.float64), _arr(head_cost, np.float64)
    sl, sa = _arr(supports_layer, np.uint8), _arr(supports_attn, np.uint8)
    mv = np.zeros(3 * max(max_moves, 1), dtype=np.int32)
    n = ctypes.c_int32()
    _check(lib().bs_plan_migrations(len(ld), ld.ctypes.data, nl.ctypes.data, ll.ctypes.data,
                                    lc.ctypes.data, nh.ctypes.data, hl.ctypes.data, hc.ctypes.data,
                                    sl.ctypes.data, sa.ctypes.data, float(delta), float(rho),
                                    int(max_moves), mv.ctypes.data, ctypes.byref(n)))
    moves = [tuple(int(v) for v in mv[3 * k:3 * k + 3]) for k in range(n.value)]
    return moves, ld.tolist(), nl.tolist(), nh.tolist()


class MigrationController:
    """Periodic control cycle with hysteresis (delta_up to start, delta_down to keep going)."""

    def __init__(self, delta_up: float, delta_down: float, rho: float):
        assert delta_down <= delta_up
        self.delta_up, self.delta_down, self.rho = delta_up, delta_down, rho
        self.active = False

    def cycle(self, load, n_layers, layer_load, layer_cost, n_heads, head_load, head_cost,
              supports_layer, supports_attn):
        delta = self.delta_down if self.active else self.delta_up
        res = plan_migrations(load, n_layers, layer_load, layer_cost, n_heads, head_load,
                              head_cost, supports_layer, supports_attn, delta, self.rho)
        self.active = bool(res[0])
        return res
