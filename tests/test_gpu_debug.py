"""Debug build (BS_DEBUG=1 -> libbanaserve_debug.so): device index arrays
are validated on the device before the launch; a violation returns BS_ERR_INVALID_ARG
without launching and sets bs_debug_error_code (1 table id, 2 kv_split vs table width,
4 migration id, 8 append position past the table).  Runs in a subprocess so the release library of the other tests is not
loaded next to the debug one."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import numpy as np, torch
import paper_2510_13223_b200 as bs
import synth
assert bs.lib().bs_debug_build() == 1
dev = torch.device("cuda", 0)
src = bs.KVPool(1, 8, 2, 64); dst = bs.KVPool(1, 8, 2, 64)
i32 = lambda x: torch.tensor(x, dtype=torch.int32, device=dev)
bs.kv_migrate_layer(src, dst, 0, i32([0, 7]), i32([1, 2]))          # valid
assert bs.lib().bs_debug_error_code(0) == 0
try:
    bs.kv_migrate_layer(src, dst, 0, i32([0, 8]), i32([1, 2]))      # src id 8 of 8 blocks
    raise SystemExit("out-of-range migration id accepted")
except bs.BSError as e:
    assert e.status == bs.BS_ERR_INVALID_ARG
assert bs.lib().bs_debug_error_code(1) == 4
shape = synth.Shape(1, 4, 2, 64)
lens = (20, 40)
dense = synth.gen_dense(shape, lens, seed=1)
ks = synth.block_aligned_split(lens, 2)
sh = synth.place_shards(dense, ks, seed=1)[0]
pool = bs.KVPool(1, sh.pool.shape[1], 2, 64)
pool.data.copy_(torch.from_numpy(sh.pool.view(np.int16)).view(torch.bfloat16).to(dev))
q = torch.from_numpy(dense.q[0].view(np.int16)).view(torch.bfloat16).to(dev)
o = torch.empty(2, 4, 64, device=dev); m = torch.empty(2, 4, device=dev); l = torch.empty(2, 4, device=dev)
bt = torch.from_numpy(sh.block_tables).to(dev)
ksd = torch.from_numpy(ks).to(dev)
ws = torch.zeros(4096, dtype=torch.uint8, device=dev)
bs.split_decode_attention(pool, 0, q, bt, ksd, 0, 0.125, o, m, l, ws)   # valid
torch.cuda.synchronize()
bad = bt.clone(); bad[1, 0] = 10_000
try:
    bs.split_decode_attention(pool, 0, q, bad, ksd, 0, 0.125, o, m, l, ws)
    raise SystemExit("out-of-range table id accepted")
except bs.BSError as e:
    assert e.status == bs.BS_ERR_INVALID_ARG
assert bs.lib().bs_debug_error_code(1) == 1
ks2 = ks.copy(); ks2[0, 1] = 16 * bt.shape[1] + 16; ks2[0, 2] = ks2[0, 1] + 1
try:
    bs.split_decode_attention(pool, 0, q, bt, torch.from_numpy(ks2).to(dev), 0, 0.125, o, m, l, ws)
    raise SystemExit("kv_split wider than the table accepted")
except bs.BSError as e:
    assert e.status == bs.BS_ERR_INVALID_ARG
assert bs.lib().bs_debug_error_code(1) & 2
# H7 append: valid, position past the table (code 8), block id out of range (code 1)
kn = torch.zeros(2, 2, 64, dtype=torch.bfloat16, device=dev)
bs.kv_append_token(pool, 0, kn, kn, bt, i32([3, -1]))
torch.cuda.synchronize()
assert bs.lib().bs_debug_error_code(0) == 0
for p, tab, code in (([16 * bt.shape[1], 0], bt, 8), ([0, 0], bad, 1)):
    try:
        bs.kv_append_token(pool, 0, kn, kn, tab, i32(p))
        raise SystemExit("invalid append accepted")
    except bs.BSError as e:
        assert e.status == bs.BS_ERR_INVALID_ARG
    assert bs.lib().bs_debug_error_code(1) == code, code
print("debug checks ok")
'''


def test_debug_build_rejects_bad_device_indices():
    env = dict(os.environ, BS_DEBUG="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "debug checks ok" in r.stdout, r.stdout + r.stderr
