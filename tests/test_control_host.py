"""Host logic of the closed F4 loop (paper_2510_13223_b200/control.py), no GPU: Cost(m)
from measured rates (eq. 35), Alg. 1's inputs derived from a module placement (eq. 32
loads, module counts), the plan bs_plan_migrations returns for them, and the head runs
attention is issued over.  The GPU execution is in tests/test_gpu_control.py."""
from types import SimpleNamespace

import pytest
import torch


@pytest.fixture(scope="module")
def control():
    import paper_2510_13223_b200 as m
    m.lib()
    from paper_2510_13223_b200 import control as c
    return c


def _placement(control, L=4, H=4, nblk=10, chunk=64 * 1024, wbytes=2**20, owner=None):
    pool = SimpleNamespace(num_layers=L, num_kv_heads=H, chunk_bytes=chunk)
    ids = torch.zeros(nblk, dtype=torch.int32)
    w = [[torch.empty(wbytes, dtype=torch.uint8) for _ in range(L)] for _ in range(2)]
    return control.ModulePlacement([pool, pool], [ids, ids], w, owner=owner)


def test_costs_are_bytes_over_measured_rate_plus_sync(control):
    c = control.MeasuredCosts(kv_layer_Bps=2e12, kv_head_Bps=1e12, weight_Bps=4e12, t_sync_s=1e-5)
    assert c.layer_cost(2e6, 4e6) == pytest.approx(1e-6 + 1e-6 + 1e-5)
    assert c.head_cost(3e6) == pytest.approx(3e-6 + 1e-5)


def test_loads_counts_and_layer_plan(control):
    pl = _placement(control)
    assert [pl.load(d) for d in range(2)] == [2.0, 0.0]
    assert pl.full_layers(0) == [0, 1, 2, 3] and pl.heads(1) == []
    c = control.MeasuredCosts(1e12, 1e12, 1e12, 1e-5)
    moves, load, n_layers, n_heads = pl.plan(c, delta=0.3, rho=1.0)
    assert moves == [(control.LAYER, 0, 1)] * 2 and load == [1.0, 1.0] and n_layers == [2, 2]


def test_expensive_layers_fall_through_to_heads(control):
    """rho between the two modules' Benefit/Cost: Alg. 1 skips the layer move (line 12)
    and takes the KV-head move (line 14)."""
    pl = _placement(control, wbytes=2**30)           # 1 GiB of weights per layer
    c = control.MeasuredCosts(1e12, 1e12, 1e12, 1e-5)
    c_layer = c.layer_cost(10 * 64 * 1024, 2**30)
    c_head = c.head_cost(4 * 10 * 2 * (64 * 1024 // 8))
    assert c_layer > c_head
    moves = pl.plan(c, delta=0.3, rho=1.0 / (c_layer * c_head) ** 0.5)[0]
    assert moves == [(control.HEADS, 0, 1)] * 2
    # with the layer path unsupported on device 0 the heads are taken at any rho it passes
    assert pl.plan(c, delta=0.3, rho=1.0, supports_layer=[0, 1])[0] == [(control.HEADS, 0, 1)] * 2
    # and nothing moves when neither passes
    assert pl.plan(c, delta=0.3, rho=1e12)[0] == []


def test_head_runs_follow_ownership(control):
    owner = [[0, 0, 1, 1], [0, 1, 1, 0], [1, 1, 1, 1], [0, 0, 0, 0]]
    pl = _placement(control, owner=owner)
    assert pl.head_runs(0) == [(0, 0, 2), (1, 2, 2)]
    assert pl.head_runs(1) == [(0, 0, 1), (1, 1, 2), (0, 3, 1)]
    assert pl.head_runs(2) == [(1, 0, 4)] and pl.head_runs(3) == [(0, 0, 4)]
    assert pl.full_layers(1) == [2] and pl.heads(1) == [0, 1, 2, 3]
    assert pl.load(0) + pl.load(1) == pytest.approx(2.0)
