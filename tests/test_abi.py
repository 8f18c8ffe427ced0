"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-side logic (geometry, allocator, argument validation,
split-K planning) behaves as documented.  No device compute is launched here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2510_13223_b200 as bs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "banaserve.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_all_exported():
    declared = header_functions()
    assert len(declared) >= 16
    assert sorted(bs.EXPORTED_SYMBOLS) == declared
    L = bs.lib()
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", bs.lib_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (bs_\w+)", out))
    assert set(declared) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", bs.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version():
    """The loaded library, the header and the binding agree on the ABI version."""
    import re
    hdr = open(os.path.join(ROOT, "include", "banaserve.h")).read()
    v = int(re.search(r"#define BS_ABI_VERSION (\d+)", hdr).group(1))
    assert bs.lib().bs_abi_version() == v == bs.ABI_VERSION


def _desc(L=2, nb=10, hkv=8, d=128, bsz=16, dtype=0, dev=0):
    return bs._Desc(L, nb, bsz, hkv, d, dtype, dev)


def test_pool_geometry_matches_oracle_and_eq15():
    L = bs.lib()
    for (nl, nb, hkv, d) in [(32, 10, 8, 128), (1, 29, 2, 64), (80, 3, 8, 128), (32, 7, 32, 128)]:
        d_ = _desc(nl, nb, hkv, d)
        assert L.bs_kv_pool_bytes(ctypes.byref(d_)) == oracle.pool_bytes(nl, nb, hkv, 16, d)
        assert L.bs_kv_chunk_bytes(ctypes.byref(d_)) == oracle.chunk_elems(hkv, 16, d) * 2
    # eq. 15: Llama-3.1-8B shape, per token per layer = chunk / 16 = 4096 B
    assert L.bs_kv_chunk_bytes(ctypes.byref(_desc(32, 1, 8, 128))) // 16 == 4096
    assert L.bs_kv_pool_bytes(ctypes.byref(_desc(d=96))) == 0
    assert L.bs_kv_pool_bytes(ctypes.byref(_desc(bsz=32))) == 0


def _create(desc, base=0x10000):
    h = ctypes.c_void_p()
    st = bs.lib().bs_kv_pool_create(ctypes.byref(desc), base, ctypes.byref(h))
    return st, h


def test_pool_create_validation():
    st, h = _create(_desc(d=96))
    assert st == bs.BS_ERR_UNSUPPORTED and not h.value
    assert b"head_dim" in bs.lib().bs_last_error()
    st, h = _create(_desc(), base=0x10010)          # misaligned
    assert st == bs.BS_ERR_INVALID_ARG
    st, h = _create(_desc(), base=0)
    assert st == bs.BS_ERR_INVALID_ARG
    st, h = _create(_desc(nb=0))
    assert st == bs.BS_ERR_INVALID_ARG
    st, h = _create(_desc())
    assert st == bs.BS_OK and h.value
    assert bs.lib().bs_kv_pool_destroy(h) == bs.BS_OK


def test_allocator_matches_oracle_policy():
    """Same random alloc/free trace on the library allocator and the oracle allocator."""
    rng = np.random.default_rng(0)
    L = bs.lib()
    for trial in range(20):
        nb = int(rng.integers(1, 64))
        st, h = _create(_desc(nb=nb))
        assert st == 0
        ref = oracle.Allocator(nb)
        live = []
        for step in range(60):
            if live and rng.random() < 0.4:
                k = int(rng.integers(1, len(live) + 1))
                idx = rng.choice(len(live), size=k, replace=False)
                ids = [live[i] for i in idx]
                buf = (ctypes.c_int32 * k)(*ids)
                assert L.bs_kv_pool_free(h, k, buf) == 0
                assert ref.free(ids)
                live = [x for i, x in enumerate(live) if i not in set(idx.tolist())]
            else:
                n = int(rng.integers(0, nb + 3))
                buf = (ctypes.c_int32 * max(n, 1))()
                st = L.bs_kv_pool_alloc(h, n, buf)
                got = ref.alloc(n)
                if got is None:
                    assert st == bs.BS_ERR_OUT_OF_BLOCKS
                else:
                    assert st == 0 and list(buf[:n]) == list(got)
                    live += list(got)
            assert L.bs_kv_pool_num_free(h) == int((ref.used == 0).sum())
        L.bs_kv_pool_destroy(h)


def test_free_errors_leave_state_unchanged():
    L = bs.lib()
    st, h = _create(_desc(nb=4))
    buf = (ctypes.c_int32 * 3)()
    assert L.bs_kv_pool_alloc(h, 3, buf) == 0
    for bad in ([0, 0], [3], [9], [-1], [1, 3]):
        b = (ctypes.c_int32 * len(bad))(*bad)
        assert L.bs_kv_pool_free(h, len(bad), b) == bs.BS_ERR_INVALID_ARG
        assert L.bs_kv_pool_num_free(h) == 1
    L.bs_kv_pool_destroy(h)


def test_launch_validation_without_device():
    """Argument errors are reported before anything is launched."""
    L = bs.lib()
    st, a = _create(_desc(L=2))
    st2, b = _create(_desc(L=3))
    ids = ctypes.c_void_p(0x1000)
    assert L.bs_kv_migrate_layer(a, b, 0, ids, ids, 1, None) == bs.BS_ERR_INVALID_ARG  # geometry
    assert L.bs_kv_migrate_layer(a, a, 2, ids, ids, 1, None) == bs.BS_ERR_INVALID_ARG  # layer
    assert L.bs_kv_migrate_layer(a, a, 0, None, ids, 1, None) == bs.BS_ERR_INVALID_ARG
    assert L.bs_kv_migrate_layer(a, a, 0, None, None, 0, None) == bs.BS_OK            # n = 0
    assert L.bs_kv_migrate_layer_ex(a, a, 0, ids, ids, 1, 7, None) == bs.BS_ERR_INVALID_ARG
    # attention: G = 3 unsupported, shard out of range, missing workspace
    p = ctypes.c_void_p(0x1000)
    f = L.bs_split_decode_attention
    assert f(a, 0, p, 4, 24, p, 8, p, 2, 2, 0.1, p, p, p, None, 0, None) == bs.BS_ERR_INVALID_ARG
    assert f(a, 0, p, 4, 12, p, 8, p, 2, 0, 0.1, p, p, p, None, 0, None) == bs.BS_ERR_INVALID_ARG
    assert f(a, 0, p, 4, 24, p, 8, p, 2, 0, float("nan"), p, p, p, None, 0, None) == bs.BS_ERR_INVALID_ARG
    assert f(a, 0, p, 4, 24, p, 8, p, 2, 0, 0.1, p, p, p, None, 0, None) == bs.BS_ERR_UNSUPPORTED
    assert b"G=3" in L.bs_last_error()
    # H7 append: NULL pool, layer out of range, NULL arrays, misaligned rows, batch 0 no-op
    ap = L.bs_kv_append_token
    assert ap(None, 0, p, p, 4, p, 8, p, None) == bs.BS_ERR_INVALID_ARG
    assert ap(a, 2, p, p, 4, p, 8, p, None) == bs.BS_ERR_INVALID_ARG
    assert ap(a, 0, p, None, 4, p, 8, p, None) == bs.BS_ERR_INVALID_ARG
    assert ap(a, 0, ctypes.c_void_p(0x1008), p, 4, p, 8, p, None) == bs.BS_ERR_INVALID_ARG
    assert ap(a, 0, p, p, 4, p, 0, p, None) == bs.BS_ERR_INVALID_ARG
    assert ap(a, 0, None, None, 0, None, 0, None, None) == bs.BS_OK
    # merge: too many parts / bad head_dim
    arr = (ctypes.c_void_p * 17)(*([0x1000] * 17))
    assert L.bs_merge_partials(17, arr, arr, arr, 1, 1, 128, p, None, None) == bs.BS_ERR_INVALID_ARG
    assert L.bs_merge_partials(2, arr, arr, arr, 1, 1, 96, p, None, None) == bs.BS_ERR_UNSUPPORTED
    L.bs_kv_pool_destroy(a)
    L.bs_kv_pool_destroy(b)


def test_split_k_workspace_plan():
    L = bs.lib()
    st, h = _create(_desc(L=1, hkv=32))
    sz = ctypes.c_size_t()
    # large batch: one CTA range per (request, kv-head), no workspace
    assert L.bs_split_decode_attention_workspace_size(h, 64, 32, 128, ctypes.byref(sz)) == 0
    assert sz.value == 0
    # B=1, 32k tokens: split-K, workspace = partials + per-(b, kv-head) counters
    L.bs_kv_pool_destroy(h)
    st, h = _create(_desc(L=1, hkv=8))
    assert L.bs_split_decode_attention_workspace_size(h, 1, 32, 2048, ctypes.byref(sz)) == 0
    assert sz.value > 0 and (sz.value - 1 * 8 * 4) % (32 * (128 + 2) * 4) == 0
    L.bs_kv_pool_destroy(h)


def test_debug_build_exports_the_same_abi():
    """libbanaserve_debug.so (-DBS_DEBUG=1) exports every declared symbol and reports
    itself as the debug build; the release library does not."""
    from paper_2510_13223_b200 import build as b
    path = b.build(debug=True)
    dbg = ctypes.CDLL(path)
    for name in header_functions():
        assert hasattr(dbg, name), name
    dbg.bs_debug_build.restype = ctypes.c_int32
    assert dbg.bs_debug_build() == 1
    assert bs.lib().bs_debug_build() == 0
    assert bs.lib().bs_debug_error_code(0) == 0


def test_package_data_plane_has_no_torch_collectives():
    """The N>1 data plane moves its bytes through the library (P2P pushes, or bs_exchange on
    the library's own NCCL communicator): torch.distributed only sets up (object gathers of
    IPC handles, the ncclUniqueId broadcast)."""
    import glob
    import re
    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2510_13223_b200")
    bad = re.compile(r"batch_isend_irecv|dist\.(all_gather|isend|irecv|send|recv|all_to_all)\(")
    for f in glob.glob(os.path.join(pkg, "*.py")):
        src = open(f).read()
        assert not bad.search(src), f


def test_ipc_export_refuses_expandable_segments(monkeypatch):
    """torch's expandable segments are virtual-memory mappings cudaIpcGetMemHandle cannot
    export: the P2P transport's ipc_export refuses that allocator mode with a clear error
    (before any CUDA call, so this runs on CPU)."""
    import torch
    import paper_2510_13223_b200 as bs
    monkeypatch.setenv("PYTORCH_CUDA_ALLOC_CONF", "max_split_size_mb:64,expandable_segments:True")
    with pytest.raises(bs.BSError, match="expandable_segments"):
        bs.ipc_export(torch.zeros(4))
    monkeypatch.setenv("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:False")
    assert not bs._expandable_segments()


def test_attention_last_launch_before_any_launch():
    """bs_attention_last_launch is host-only: all zeros before the thread's first launch,
    BS_ERR_INVALID_ARG on a NULL output."""
    import ctypes
    info = bs.attention_last_launch()
    assert info == {"ranges": 0, "merge": 0, "pdl": 0, "tensor_cores": 0, "stages": 0, "cluster": 0}
    v = ctypes.c_int32()
    st = bs.lib().bs_attention_last_launch(None, ctypes.byref(v), ctypes.byref(v), ctypes.byref(v),
                                           ctypes.byref(v))
    assert st == bs.BS_ERR_INVALID_ARG


def test_ragged_plan_ex_rejects_unknown_flags():
    import ctypes
    ks = np.array([[0, 100]], dtype=np.int32)
    sa = (ctypes.c_int32 * 1)(0)
    nw, mp, wsb = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_size_t()
    st = bs.lib().bs_attention_ragged_plan_ex(1, 1, ks.ctypes.data, 1, sa, 8, 2, 128, 0, 0x80,
                                              None, 0, ctypes.byref(nw), ctypes.byref(mp),
                                              ctypes.byref(wsb))
    assert st == bs.BS_ERR_INVALID_ARG
