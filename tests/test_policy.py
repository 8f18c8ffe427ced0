"""NEXT row F4 (control plane): the oracle (oracle/policy.py) pinned to
hand-worked runs of Alg. 1 / Alg. 2 and to invariants, and the product's C++ policy
(bs_dispatch_requests / bs_plan_migrations) equal to the oracle on random instances.
CPU only."""
import random

import pytest

from oracle import policy as ref
from paper_2510_13223_b200 import policy as prod


# ------------------------------------------------------------------ oracle pins (Alg. 2)

def test_alg2_hand_worked_least_loaded():
    # loads [0.5, 0.2, 0.9], queues [3, 1, 0], delta_L = 0.6, three requests of 0.3:
    # r0 -> 1 (0.2 < 0.6; load 0.5, q 2); r1 -> 1 ((0.5,2,1) < (0.5,3,0); load 0.8, q 3);
    # r2 -> 0 (0.5 < 0.6; load 0.8, q 4)
    assign, load, q = ref.dispatch([0.5, 0.2, 0.9], [3, 1, 0], [0.3, 0.3, 0.3], 0.6)
    assert assign == [1, 1, 0]
    assert load == pytest.approx([0.8, 0.8, 0.9]) and q == [4, 3, 0]


def test_alg2_hand_worked_lowest_queue():
    # every instance at/above delta_L: lines 16-18 pick the lowest queue, loads unchanged
    assign, load, q = ref.dispatch([0.9, 0.8], [2, 5], [0.1] * 4, 0.6)
    assert assign == [0, 0, 0, 1]            # queues 3,4,5 then tie (5,0.9,0) vs (5,0.8,1)
    assert load == [0.9, 0.8] and q == [5, 6]


def test_utilization_eq32_range():
    assert ref.utilization(0, 1, 0, 1) == 0.0
    assert ref.utilization(1, 1, 1, 1) == 2.0
    assert ref.utilization(35, 100, 95, 100) == pytest.approx(1.3)


# ------------------------------------------------------------------ oracle pins (Alg. 1)

def _dev(n, layers=4, heads=8, lu=0.2, lc=1.0, hu=0.05, hc=0.1, sl=1, sa=1):
    return dict(n_layers=[layers] * n, layer_load=[lu] * n, layer_cost=[lc] * n,
                n_heads=[heads] * n, head_load=[hu] * n, head_cost=[hc] * n,
                supports_layer=[sl] * n, supports_attn=[sa] * n)


def test_alg1_hand_worked_layer_moves():
    # loads [1.6, 0.4], delta 0.3, layer share 0.2: gaps 1.2 -> 0.8 -> 0.4 -> 0.0
    moves, load, nl, nh = ref.plan_migrations([1.6, 0.4], delta=0.3, rho=0.1, **_dev(2))
    assert moves == [(0, 0, 1)] * 3
    assert load == pytest.approx([1.0, 1.0]) and nl == [1, 7] and nh == [8, 8]


def test_alg1_rho_gate_and_fallback_to_heads():
    # layer moves cost 100 s: benefit/cost < rho -> fall through to KV-head moves (0.05)
    moves, load, _, _ = ref.plan_migrations([1.0, 0.7], delta=0.1, rho=0.5,
                                            **_dev(2, lc=100.0))
    assert moves and all(k == 1 for k, _, _ in moves)
    assert max(load) - min(load) <= 0.1 + 1e-12
    # nothing passes the gate -> no move at all
    moves, load, _, _ = ref.plan_migrations([1.0, 0.7], delta=0.1, rho=0.5,
                                            **_dev(2, lc=100.0, hc=100.0))
    assert moves == [] and load == [1.0, 0.7]


def test_alg1_overshoot_rejected():
    # a 0.5-layer would overshoot a 0.4 gap (benefit 0.4 - 0.6 < 0) -> heads instead
    moves, load, _, _ = ref.plan_migrations([0.9, 0.5], delta=0.3, rho=0.01,
                                            **_dev(2, lu=0.5, hu=0.1))
    assert moves[0][0] == 1 and load == pytest.approx([0.8, 0.6])


def test_alg1_invariants_random():
    rng = random.Random(0)
    for _ in range(300):
        D = rng.randint(2, 9)
        load = [rng.uniform(0, 2) for _ in range(D)]
        kw = dict(n_layers=[rng.randint(0, 5) for _ in range(D)],
                  layer_load=[rng.uniform(0.01, 0.4) for _ in range(D)],
                  layer_cost=[rng.uniform(0.1, 3) for _ in range(D)],
                  n_heads=[rng.randint(0, 8) for _ in range(D)],
                  head_load=[rng.uniform(0.005, 0.1) for _ in range(D)],
                  head_cost=[rng.uniform(0.01, 1) for _ in range(D)],
                  supports_layer=[rng.randint(0, 1) for _ in range(D)],
                  supports_attn=[rng.randint(0, 1) for _ in range(D)])
        delta, rho = rng.uniform(0.05, 0.5), rng.uniform(0, 0.5)
        moves, out, nl, nh = ref.plan_migrations(load, delta=delta, rho=rho, **kw)
        assert sum(out) == pytest.approx(sum(load))                     # conservation
        assert sum(nl) == sum(kw["n_layers"]) and sum(nh) == sum(kw["n_heads"])
        assert max(out) <= max(load) + 1e-12                            # never worse
        # termination condition: no (overload, underload) pair with a passing move
        again, _, _, _ = ref.plan_migrations(out, delta=delta, rho=rho,
                                             **dict(kw, n_layers=nl, n_heads=nh))
        assert again == []


# ------------------------------------------------------------------ product == oracle

def test_product_dispatch_equals_oracle():
    rng = random.Random(1)
    for _ in range(300):
        P = rng.randint(1, 12)
        load = [round(rng.uniform(0, 2), 3) for _ in range(P)]
        q = [rng.randint(0, 6) for _ in range(P)]
        est = [round(rng.uniform(0, 0.3), 3) for _ in range(rng.randint(0, 40))]
        dl = rng.uniform(0.2, 1.8)
        assert prod.dispatch(load, q, est, dl) == ref.dispatch(load, q, est, dl)


def test_product_plan_equals_oracle():
    rng = random.Random(2)
    for _ in range(300):
        D = rng.randint(1, 10)
        load = [rng.uniform(0, 2) for _ in range(D)]
        kw = dict(n_layers=[rng.randint(0, 5) for _ in range(D)],
                  layer_load=[rng.uniform(0.01, 0.4) for _ in range(D)],
                  layer_cost=[rng.uniform(0.1, 3) for _ in range(D)],
                  n_heads=[rng.randint(0, 8) for _ in range(D)],
                  head_load=[rng.uniform(0.005, 0.1) for _ in range(D)],
                  head_cost=[rng.uniform(0.01, 1) for _ in range(D)],
                  supports_layer=[rng.randint(0, 1) for _ in range(D)],
                  supports_attn=[rng.randint(0, 1) for _ in range(D)])
        delta, rho = rng.uniform(0.05, 0.5), rng.uniform(0, 0.5)
        got = prod.plan_migrations(load, delta=delta, rho=rho, **kw)
        exp = ref.plan_migrations(load, delta=delta, rho=rho, **kw)
        assert got[0] == exp[0] and got[1] == exp[1] and got[2] == exp[2] and got[3] == exp[3]


def test_hysteresis_controller():
    c = prod.MigrationController(delta_up=0.5, delta_down=0.1, rho=0.01)
    kw = _dev(2, lu=0.1, hu=0.02)
    # gap 0.4 < delta_up: idle controller does nothing
    moves, load, nl, nh = c.cycle([1.0, 0.6], **kw)
    assert moves == [] and not c.active
    # gap 0.8 > delta_up: the cycle starts migrating (classified with delta_up) ...
    moves, load, nl, nh = c.cycle([1.2, 0.4], **kw)
    assert moves and c.active and 0.1 < max(load) - min(load) <= 0.5 + 1e-12
    # ... and the next cycles keep going down to delta_down, then go idle
    moves, load, nl, nh = c.cycle(load, **dict(kw, n_layers=nl, n_heads=nh))
    assert moves and max(load) - min(load) <= 0.1 + 1e-12
    moves, load, nl, nh = c.cycle(load, **dict(kw, n_layers=nl, n_heads=nh))
    assert moves == [] and not c.active
    assert prod.utilization(35, 100, 95, 100) == pytest.approx(1.3)


def test_oracle_hysteresis_hand_worked():
    """R-F4g, worked by hand with exactly representable numbers: delta_up =
    1/4, delta_down = 1/8, one layer carries 1/16 of load (cost 1, rho 0.1).
      cycle 1 (idle -> delta_up):   [1, 1/2]: gap 1/2 > 1/4 -> move -> [15/16, 9/16]:
                                    gap 3/8 > 1/4 -> move -> [7/8, 5/8]: gap 1/4, stop (2 moves)
      cycle 2 (migrating -> delta_down): gap 1/4 > 1/8 -> move -> [13/16, 11/16]: stop (1)
      cycle 3 (migrating -> delta_down): gap 1/8, no move -> idle
      cycle 4 (idle -> delta_up): new loads [7/8, 11/16], gap 3/16 -- above delta_down but
                                    not delta_up: no move (the hysteresis band)
      cycle 5 (idle): [1, 11/16], gap 5/16 > 1/4 -> move -> [15/16, 3/4]: gap 3/16, stop."""
    kw = _dev(2, layers=4, lu=1 / 16, lc=1.0, sa=0)
    cycles = []
    for ld in ([1.0, 0.5], None, None, [0.875, 0.6875], [1.0, 0.6875]):
        if cycles:   # the next period starts from the placement the last one left
            prev = ref.run_cycles(cycles, 0.25, 0.125, 0.1)[-1]
            kw = dict(kw, n_layers=prev[2], n_heads=prev[3])
            ld = prev[1] if ld is None else ld
        cycles.append(dict(kw, load=ld))
    got = ref.run_cycles(cycles, 0.25, 0.125, 0.1)
    assert [len(r[0]) for r in got] == [2, 1, 0, 0, 1]
    assert got[0][1] == [0.875, 0.625] and got[1][1] == [0.8125, 0.6875]
    assert got[2][1] == [0.8125, 0.6875] and got[3][1] == [0.875, 0.6875]
    assert got[4][1] == [0.9375, 0.75]
    # without hysteresis (delta_up = delta_down = 1/8) cycle 4 would have moved
    flat = ref.run_cycles(cycles, 0.125, 0.125, 0.1)
    assert len(flat[3][0]) == 1


def test_product_controller_equals_oracle_hysteresis():
    """MigrationController (product) == oracle.run_cycles on random cycle sequences."""
    rng = random.Random(5)
    for _ in range(100):
        D = rng.randint(2, 6)
        up = rng.uniform(0.15, 0.5)
        down = rng.uniform(0.02, up)
        rho = rng.uniform(0, 0.3)
        c = prod.MigrationController(up, down, rho)
        tables = dict(layer_load=[rng.uniform(0.01, 0.3) for _ in range(D)],
                      layer_cost=[rng.uniform(0.1, 2) for _ in range(D)],
                      head_load=[rng.uniform(0.005, 0.08) for _ in range(D)],
                      head_cost=[rng.uniform(0.01, 1) for _ in range(D)],
                      supports_layer=[rng.randint(0, 1) for _ in range(D)],
                      supports_attn=[1] * D)
        nl, nh = [rng.randint(0, 5) for _ in range(D)], [rng.randint(0, 8) for _ in range(D)]
        cyc = []
        for _ in range(rng.randint(1, 8)):
            load = [rng.uniform(0, 2) for _ in range(D)]
            cyc.append(dict(tables, load=load, n_layers=list(nl), n_heads=list(nh)))
            got = c.cycle(load, n_layers=nl, n_heads=nh, **tables)
            nl, nh = got[2], got[3]
            exp = ref.run_cycles(cyc, up, down, rho)[-1]
            assert got[0] == exp[0] and got[1] == exp[1] and got[2] == exp[2] and got[3] == exp[3]
