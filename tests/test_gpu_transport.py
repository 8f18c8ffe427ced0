"""GPU tests of the cross-instance transports on ONE GPU (the only topology gpurun offers):
  * NCCL two-sided H2 (bs_kv_sendrecv_layer, bs_kv_send/recv_layer) and the H5 partial
    exchange (bs_sendrecv) over a 1-rank communicator, loopback;
  * CUDA IPC remote views: a second process maps the first one's pool and pushes chunks
    into it with bs_kv_migrate_layer (the P2P-push code path; over NVLink when the two
    processes own different GPUs).
Expected values come from the oracle's migrate (bit-exact)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu


def _rand_pool(shape, nb, L, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 65536, (L, nb, 2, shape.hkv, 16, shape.d), generator=g,
                         dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)


def _to_pool(bs, arr, shape):
    p = bs.KVPool(arr.shape[0], arr.shape[1], shape.hkv, shape.d)
    p.data.copy_(torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16).cuda())
    return p


def _u16(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.fixture(scope="module")
def bs():
    import paper_2510_13223_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="module")
def comm(bs):
    c = bs.Comm(bs.nccl_unique_id(), 1, 0)
    yield c
    c.close()


def test_nccl_loopback_kv_sendrecv_layer(bs, comm):
    shape = synth.Shape(2, 8, 8, 128)
    src_np = _rand_pool(shape, 40, 2, 1)
    dst_np = np.full((2, 50, 2, 8, 16, 128), synth.DST_SENTINEL, dtype=np.uint16)
    src, dst = _to_pool(bs, src_np, shape), _to_pool(bs, dst_np, shape)
    s = np.array([5, 0, 39, 17], dtype=np.int32)
    t = np.array([49, 3, 2, 20], dtype=np.int32)
    st_s = torch.empty(len(s) * src.chunk_bytes, dtype=torch.uint8, device="cuda")
    st_r = torch.empty_like(st_s)
    si, ti = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
    bs.kv_sendrecv_layer(comm, src, si, 0, st_s, dst, ti, 0, st_r, 1)
    torch.cuda.synchronize()
    ref = dst_np.copy()
    oracle.migrate_layer(src_np, ref, 1, s, t)
    assert np.array_equal(_u16(dst.data), ref)


def test_nccl_partial_exchange_bytes(bs, comm):
    send = torch.randn(64 * 32 * 130, device="cuda")
    recv = torch.zeros_like(send)
    comm.sendrecv(send, 0, recv, 0)
    torch.cuda.synchronize()
    assert torch.equal(send, recv)


def _ipc_child(handle, offset, shape_t, L, nb, src_bytes, s, t, q):
    try:
        import paper_2510_13223_b200 as bsm
        torch.cuda.set_device(0)
        shape = synth.Shape(*shape_t)
        ptr = bsm.ipc_import(handle, offset)
        # remote view of the parent's pool, described by the raw peer-mapped pointer
        desc = bsm._Desc(L, nb, 16, shape.hkv, shape.d, 0, 0)
        import ctypes
        h = ctypes.c_void_p()
        bsm._check(bsm.lib().bs_kv_pool_create(ctypes.byref(desc), ptr, ctypes.byref(h)))

        class _View:
            handle = h
        src_np = np.frombuffer(src_bytes, dtype=np.uint16).reshape(L, nb, 2, shape.hkv, 16, shape.d)
        src = _to_pool(bsm, src_np.copy(), shape)
        bsm.kv_migrate_layer(src, _View, 1, torch.tensor(s, dtype=torch.int32, device="cuda"),
                             torch.tensor(t, dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
        bsm.lib().bs_kv_pool_destroy(h)
        bsm.ipc_close(ptr, offset)
        q.put("ok")
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(traceback.format_exc())


def test_ipc_remote_view_push(bs):
    shape = synth.Shape(2, 4, 4, 128)
    L, nb = 2, 30
    dst_np = np.full((L, nb, 2, 4, 16, 128), synth.DST_SENTINEL, dtype=np.uint16)
    dst = _to_pool(bs, dst_np, shape)
    # export an interior pointer: the layer-0 offset exercises the handle+offset path
    handle, offset = bs.ipc_export(dst.data)
    src_np = _rand_pool(shape, nb, L, 7)
    s = [1, 2, 29, 0]
    t = [0, 28, 5, 6]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ipc_child, args=(handle, offset, (2, 4, 4, 128), L, nb,
                                             src_np.tobytes(), s, t, q))
    p.start()
    msg = q.get(timeout=300)
    p.join(timeout=60)
    assert msg == "ok", msg
    ref = dst_np.copy()
    oracle.migrate_layer(src_np, ref, 1, np.array(s, dtype=np.int32), np.array(t, dtype=np.int32))
    assert np.array_equal(_u16(dst.data), ref)
