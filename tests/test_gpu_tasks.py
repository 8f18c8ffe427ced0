"""bs_split_decode_attention_tasks (H4 + H5 + H6 fused across launches, SURVEY.md §8(e)
"fused B200 variant"): attention problems whose shards are processed by DIFFERENT
launches -- stand-ins for different GPUs, each on its own stream so they run
concurrently on GPU 0 -- write their partials into the problem's workspace, and the
last-arriving CTA (from whichever launch) merges into the home buffers.  Checked against
the oracle (attention over the request's whole KV), against the single-launch fused path
(bitwise: same range plan, same fixed merge order), and for the `done` counter."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ABS_TOL, ROW_REL_TOL, LSE_TOL = 2e-2, 1e-2, 1e-4


@pytest.fixture(scope="module")
def bs():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2510_13223_b200 as m
    m.lib()
    return m


def dev_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def dev_i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


class Problem:
    def __init__(self, bs, shape, lens, n_shards, seed, cross_device):
        self.shape, self.lens = shape, lens
        self.dense = synth.gen_dense(shape, lens, seed=seed)
        self.ks = synth.random_split(lens, n_shards, seed=seed)
        self.shards = synth.place_shards(self.dense, self.ks, seed=seed)
        self.pools = []
        for s in self.shards:
            p = bs.KVPool(shape.n_layers, s.pool.shape[1], shape.hkv, shape.d)
            p.data.copy_(dev_bf16(s.pool))
            self.pools.append(p)
        self.bts = [dev_i32(s.block_tables) for s in self.shards]
        self.max_blocks = [t.shape[1] for t in self.bts]
        B, L = len(lens), shape.n_layers
        n = bs.attention_problem_workspace_size(B, shape.hq, shape.hkv, shape.d, self.max_blocks)
        self.ws = [torch.zeros(max(n, 16), dtype=torch.uint8, device="cuda") for _ in range(L)]
        self.q = dev_bf16(self.dense.q)
        self.ksd = dev_i32(self.ks)
        self.out = torch.full((L, B, shape.hq, shape.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        self.lse = torch.full((L, B, shape.hq), float("nan"), device="cuda")
        self.done = torch.zeros(L, dtype=torch.int32, device="cuda")
        self.cross_device = cross_device

    def desc(self, layer):
        return {"q": self.q[layer], "kv_split": self.ksd, "max_blocks": self.max_blocks,
                "out": self.out[layer], "lse": self.lse[layer], "workspace": self.ws[layer],
                "done": self.done[layer:layer + 1], "cross_device": self.cross_device}

    def check(self, layer):
        sc = synth.default_scale(self.shape.d)
        ref_o, ref_lse = oracle.attention_full([s.pool for s in self.shards],
                                               [s.block_tables for s in self.shards], layer,
                                               self.dense.q[layer], self.ks, sc)
        got = self.out[layer].float().cpu().double().numpy()
        gl = self.lse[layer].cpu().double().numpy()
        fin = np.isfinite(ref_lse)
        assert np.array_equal(np.isneginf(gl), ~fin) and np.all(got[~fin] == 0)
        err = np.abs(got - ref_o)
        assert err.max() <= ABS_TOL
        assert (err.max(-1)[fin] / np.abs(ref_o).max(-1)[fin]).max() <= ROW_REL_TOL
        assert np.abs(gl[fin] - ref_lse[fin]).max() <= LSE_TOL


@pytest.mark.parametrize("d,G,n_shards,cross", [(128, 1, 2, True), (128, 4, 2, False),
                                                (128, 8, 3, True), (64, 2, 4, False),
                                                (128, 1, 4, True)])
def test_two_problems_sharded_over_concurrent_launches(bs, d, G, n_shards, cross):
    shape = synth.Shape(2, 2 * G, 2, d)
    A = Problem(bs, shape, (0, 1, 17, 100, 700, 2000), n_shards, seed=d + G, cross_device=cross)
    Bp = Problem(bs, shape, (5, 2000, 64, 0, 333, 48), n_shards, seed=d + G + 1, cross_device=cross)
    B = len(A.lens)
    sc = synth.default_scale(d)
    streams = [torch.cuda.Stream() for _ in range(n_shards)]
    first = None
    for epoch in range(2):
        torch.cuda.synchronize()
        for layer in range(shape.n_layers):
            for i, st in enumerate(streams):
                # "GPU" i: shard i of A (home A) and shard n-1-i of B (home B)
                j = n_shards - 1 - i
                bs.split_decode_attention_tasks(
                    [A.desc(layer), Bp.desc(layer)],
                    [(A.pools[i], A.bts[i], i, 0), (Bp.pools[j], Bp.bts[j], j, 1)],
                    layer, B, shape.hq, sc, stream=st)
        torch.cuda.synchronize()
        for P in (A, Bp):
            assert P.done.tolist() == [(epoch + 1) * B * shape.hkv] * shape.n_layers
            for layer in range(shape.n_layers):
                P.check(layer)
        snap = (A.out.clone(), Bp.out.clone())
        if first is None:
            first = snap
        else:  # fixed merge order: bitwise reproducible whichever launch merged
            assert torch.equal(first[0].view(torch.int16), snap[0].view(torch.int16))
            assert torch.equal(first[1].view(torch.int16), snap[1].view(torch.int16))
    # same result as the single-launch fused path over the same shards (same plan)
    ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
        A.pools, A.max_blocks, B, shape.hq)), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(A.out[0])
    bs.split_decode_attention_local(A.pools, 1, A.q[1], A.bts, list(range(n_shards)), A.ksd, sc,
                                    out, None, ws)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), A.out[1].view(torch.int16))


@pytest.mark.parametrize("n_shards", [1, 3])
def test_task_request_order_changes_dispatch_not_results(bs, n_shards):
    """bs_attn_task.order (ABI 2): CTA row z serves request order[z] -- the sequence-sharded
    step passes longest-shard-first -- and the outputs are bitwise those of the identity
    order (the merge follows the range slots), and match the oracle."""
    shape = synth.Shape(2, 16, 2, 128)
    lens = (0, 3000, 17, 700, 2048, 1, 5000, 64)
    A = Problem(bs, shape, lens, n_shards, seed=21, cross_device=False)
    B = len(lens)
    sc = synth.default_scale(128)
    sh = (A.ks[:, 1:] - A.ks[:, :-1])
    orders = [dev_i32(np.argsort(-sh[:, j], kind="stable")) for j in range(n_shards)]
    outs = []
    for use_order in (False, True):
        A.out.fill_(float("nan"))
        for layer in range(shape.n_layers):
            bs.split_decode_attention_tasks(
                [A.desc(layer)],
                [(A.pools[j], A.bts[j], j, 0, orders[j] if use_order else None) for j in range(n_shards)],
                layer, B, shape.hq, sc)
        torch.cuda.synchronize()
        outs.append((A.out.clone(), A.lse.clone()))
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1], outs[1][1])
    for layer in range(shape.n_layers):
        A.check(layer)


def test_tasks_argument_errors(bs):
    shape = synth.Shape(1, 4, 2, 64)
    A = Problem(bs, shape, (10, 40), 2, seed=3, cross_device=False)
    d0 = A.desc(0)
    with pytest.raises(bs.BSError):   # shard id outside the problem
        bs.split_decode_attention_tasks([d0], [(A.pools[0], A.bts[0], 2, 0)], 0, 2, 4, 0.125)
    with pytest.raises(bs.BSError):   # problem index outside the list
        bs.split_decode_attention_tasks([d0], [(A.pools[0], A.bts[0], 0, 1)], 0, 2, 4, 0.125)
    bad = dict(d0, workspace=None, workspace_bytes=0)
    with pytest.raises(bs.BSError):   # a 2-shard problem needs its workspace
        bs.split_decode_attention_tasks([bad], [(A.pools[0], A.bts[0], 0, 0)], 0, 2, 4, 0.125)


@pytest.mark.parametrize("seed", range(12))
def test_tasks_fuzz(bs, seed):
    """Random shapes, lengths (incl. empty), unaligned splits, 1-4 shards per problem and a
    random assignment of the shards of two problems to 1-3 concurrent launches."""
    rng = np.random.default_rng(100 + seed)
    G = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 128]))
    n_shards = int(rng.integers(1, 5))
    B = int(rng.integers(1, 9))
    shape = synth.Shape(1, 2 * G, 2, d)
    lens_a = tuple(int(x) for x in rng.integers(0, 1500, B))
    lens_b = tuple(int(x) for x in rng.integers(0, 1500, B))
    A = Problem(bs, shape, lens_a, n_shards, seed=seed, cross_device=bool(seed % 2))
    Bp = Problem(bs, shape, lens_b, n_shards, seed=seed + 50, cross_device=bool(seed % 2))
    n_launch = int(rng.integers(1, 4))
    owner = [(int(rng.integers(0, n_launch)), int(rng.integers(0, n_launch))) for _ in range(n_shards)]
    sc = synth.default_scale(d)
    streams = [torch.cuda.Stream() for _ in range(n_launch)]
    torch.cuda.synchronize()
    for li, st in enumerate(streams):
        tasks = [(A.pools[j], A.bts[j], j, 0) for j in range(n_shards) if owner[j][0] == li]
        tasks += [(Bp.pools[j], Bp.bts[j], j, 1) for j in range(n_shards) if owner[j][1] == li]
        if tasks:
            bs.split_decode_attention_tasks([A.desc(0), Bp.desc(0)], tasks, 0, B, shape.hq, sc,
                                            stream=st)
    torch.cuda.synchronize()
    for P in (A, Bp):
        assert P.done[0].item() == B * shape.hkv
        P.check(0)
