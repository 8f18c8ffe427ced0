"""Host logic of the ragged plan (bs_attention_ragged_plan, no GPU): every non-empty
(request, local shard) is covered by contiguous ranges of <= max_blocks_per_range blocks,
exactly once; empty shards get no CTA; an all-empty request gets one empty item; slots
0..parts-1 per request in shard-major order; the workspace size follows max_parts."""
import numpy as np
import pytest

import synth


@pytest.fixture(scope="module")
def bs():
    import paper_2510_13223_b200 as m
    m.lib()
    return m


def check_plan(plan, ks, shard_ids, bps, hq, hkv, d):
    B = ks.shape[0]
    w = plan.work
    seen = {}
    for b, ts, blo, nbp in w:
        t, slot = ts >> 16, ts & 0xFFFF
        nb, parts = nbp >> 8, nbp & 0xFF
        seen.setdefault(int(b), []).append((int(t), int(slot), int(blo), int(nb), int(parts)))
    assert sorted(seen) == list(range(B))
    # dispatch order: longest range first
    nbs = [int(x) >> 8 for x in w[:, 3]]
    assert nbs == sorted(nbs, reverse=True)
    most = 1
    for b, items in seen.items():
        items.sort(key=lambda x: x[1])  # by slot
        nblk = [-(-max(int(ks[b, j + 1] - ks[b, j]), 0) // 16) for j in shard_ids]
        parts = {p for *_, p in items}
        assert len(parts) == 1
        p = parts.pop()
        if sum(nblk) == 0:
            assert items == [(0, 0, 0, 0, 1)]
            continue
        assert p == len(items) and [s for _, s, *_ in items] == list(range(p))
        most = max(most, p)
        # shard-major order, contiguous cover of each shard's blocks, ranges <= bps
        assert [t for t, *_ in items] == sorted(t for t, *_ in items)
        for t, n in enumerate(nblk):
            rs = [(blo, nb) for tt, _, blo, nb, _ in items if tt == t]
            assert sum(nb for _, nb in rs) == n
            pos = 0
            for blo, nb in rs:
                assert blo == pos and 1 <= nb <= bps
                pos += nb
    assert plan.max_parts == most
    exp_ws = 0 if most == 1 else B * hq * most * (d + 2) * 4 + B * hkv * 4
    assert plan.workspace_bytes == exp_ws


@pytest.mark.parametrize("bps", [16, 64, 512])
def test_ragged_plan_mixed_lengths(bs, bps):
    lens = synth.mixed_lengths(256, seed=0)
    ks = synth.block_aligned_split(lens, 8)
    plan = bs.attention_ragged_plan(ks, [2, 5], 64, 8, 128, max_blocks_per_range=bps)
    check_plan(plan, ks, [2, 5], bps, 64, 8, 128)


def test_ragged_plan_empty_and_single(bs):
    ks = np.array([[0, 0, 0], [0, 5, 5], [0, 0, 300], [0, 4096, 8192]], dtype=np.int32)
    plan = bs.attention_ragged_plan(ks, [0, 1], 32, 8, 128, max_blocks_per_range=32)
    check_plan(plan, ks, [0, 1], 32, 32, 8, 128)
    assert plan.n_work == 1 + 1 + 1 + 16


def test_ragged_plan_caps_ranges_per_request(bs):
    ks = np.array([[0, 32768 * 4]], dtype=np.int32)   # 8192 blocks: 16-block ranges would be 512
    plan = bs.attention_ragged_plan(ks, [0], 32, 8, 128, max_blocks_per_range=16)
    assert plan.max_parts <= 64
    check_plan(plan, ks, [0], 512, 32, 8, 128)


def test_ragged_plan_auto_range(bs):
    ks = synth.block_aligned_split(np.full(64, 2048), 2)
    plan = bs.attention_ragged_plan(ks, [0, 1], 32, 32, 128)    # C2: one range per shard
    assert plan.n_work == 128 and plan.max_parts == 2


def test_ragged_plan_packs_short_requests(bs):
    """pack_short (one local shard): requests of <= 8 blocks go four to an item -- parts
    field 0, (b0, b1, b2, b3 << 8), -1 = none -- every request exactly once overall, the
    others as in the plain plan; dispatch order by the CTA's longest per-warp run."""
    lens = synth.mixed_lengths(256, seed=0)
    ks = synth.block_aligned_split(lens, 8)
    plain = bs.attention_ragged_plan(ks, [3], 64, 8, 128)
    packed = bs.attention_ragged_plan(ks, [3], 64, 8, 128, pack_short=True)
    nblk = -(-(ks[:, 4] - ks[:, 3]) // 16)
    short = set(int(b) for b in np.nonzero(nblk <= 8)[0])
    assert len(short) > 50          # the Alpaca-like half
    seen, keys = [], []
    for x, y, z, w in packed.work:
        if (w & 0xFF) == 0:
            reqs = [int(v) for v in (x, y, z, w >> 8) if v >= 0]
            assert reqs and all(r in short for r in reqs)
            seen += reqs
            keys.append(4 * max(int(nblk[r]) for r in reqs))
        else:
            assert int(x) not in short
            seen.append(int(x))
            keys.append(int(w) >> 8)
    assert sorted(seen) == sorted(set(seen)) == list(range(256))
    assert keys == sorted(keys, reverse=True)
    # the unpacked requests are cut exactly as in the plain plan
    norm = sorted(tuple(int(v) for v in r) for r in packed.work if (r[3] & 0xFF) != 0)
    ref = sorted(tuple(int(v) for v in r) for r in plain.work if int(r[0]) not in short)
    assert norm == ref
    assert packed.n_work == len(ref) + -(-len(short) // 4)


def test_ragged_plan_no_packing_with_several_shards(bs):
    ks = synth.block_aligned_split(np.array([20, 3000, 50, 7]), 2)
    a = bs.attention_ragged_plan(ks, [0, 1], 32, 8, 128)
    b = bs.attention_ragged_plan(ks, [0, 1], 32, 8, 128, pack_short=True)
    assert np.array_equal(a.work, b.work)
