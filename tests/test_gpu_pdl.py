"""Programmatic dependent launch of the fused local attention (BS_ATTN_PDL: multi-wave
launches and launches of at most one CTA per SM): consecutive layers' launches on one stream share one split-K workspace, each
prefetching its K/V while the previous one drains and touching q / outputs / workspace only
after griddepcontrol.wait.  The outputs must equal the plain launches bit for bit (same plan,
same merge order) and the oracle within the north-star tolerances -- eagerly and replayed
from a CUDA graph."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bs():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2510_13223_b200 as m
    m.lib()
    return m


CASES = {
    # multi-wave (C2-like MHA, 2 local shards): the next grid starts once every CTA started
    "multiwave": (synth.Shape(4, 32, 32, 128), np.full(64, 600), 2, [0, 31, 63]),
    # one CTA per SM (C3 B=1 GQA-4, split-K 16 ranges): starts once every CTA's loop is done
    "one_per_sm": (synth.Shape(4, 32, 8, 128), np.full(1, 8192), 1, [0]),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_pdl_layers_bitwise_equal_plain_and_oracle(bs, graph, name):
    shape, lens, n_shards, sample = CASES[name]
    ks = synth.block_aligned_split(lens, n_shards)
    case = synth.device_shards(shape, lens, ks, seed=13, device="cuda")
    pools = [bs.KVPool(shape.n_layers, p.shape[1], shape.hkv, shape.d, base=p.reshape(-1))
             for p in case.pools]
    bts = [torch.from_numpy(b).cuda() for b in case.block_tables]
    ksd = torch.from_numpy(ks).cuda()
    sc = synth.default_scale(shape.d)
    B, L = len(lens), shape.n_layers
    ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
        pools, [t.shape[1] for t in bts], B, shape.hq)), dtype=torch.uint8, device="cuda")

    infos = []

    def run(flags):
        out = torch.full((L, B, shape.hq, shape.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        lse = torch.full((L, B, shape.hq), float("nan"), device="cuda")

        def step():
            for layer in range(L):
                bs.split_decode_attention_local(pools, layer, case.q[layer], bts,
                                                list(range(n_shards)), ksd, sc,
                                                out[layer], lse[layer], ws,
                                                flags=flags if layer else 0)
                if layer:
                    infos.append(bs.attention_last_launch())
        if graph:
            step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            out.fill_(float("nan"))
            g.replay()
        else:
            step()
        torch.cuda.synchronize()
        return out, lse

    o0, l0 = run(0)
    assert all(i["pdl"] == 0 for i in infos)
    infos.clear()
    o1, l1 = run(bs.ATTN_PDL)
    assert infos and all(i["pdl"] == 1 for i in infos), infos
    if name == "one_per_sm":   # the 6-stage ring: the prefetch before griddepcontrol.wait
        assert all(i["stages"] == 6 for i in infos), infos
    assert torch.equal(o0.view(torch.int16), o1.view(torch.int16))
    assert torch.equal(l0, l1)
    for layer in (0, L - 1):
        sp, sbt, sks, sq = synth.extract_requests(case, sample, layer)
        ref_o, ref_lse = oracle.attention_full(sp, sbt, 0, sq, sks, sc)
        got = o1[layer, sample].float().cpu().double().numpy()
        assert np.abs(got - ref_o).max() <= 2e-2
        assert np.abs(l1[layer, sample].cpu().double().numpy() - ref_lse).max() <= 1e-4
