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


def test_nccl_exchange_grouped_loopback(bs, comm):
    """bs_exchange: several sends / receives of different sizes in one NCCL group."""
    sends = [torch.randn(n, device="cuda") for n in (1, 4097, 300000)]
    recvs = [torch.zeros_like(t) for t in sends]
    comm.exchange([(t, 0) for t in sends], [(t, 0) for t in recvs])
    torch.cuda.synchronize()
    for a, b in zip(sends, recvs):
        assert torch.equal(a, b)


def test_wait_signal_is_wrap_safe(bs):
    """Flags and `done` counters are int32 and wrap after 2^31 (a long-running server):
    a wait whose target wrapped past INT32_MAX is satisfied by the wrapped flag value and
    not by an older one."""
    from paper_2510_13223_b200.transport import ErrorFlag
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = ErrorFlag()
    big = 2 ** 31 - 3
    flag.fill_(bs.wrap_i32(big + 5))              # 2^31 + 2 wrapped to a negative int32
    bs.wait_signal(flag.data_ptr(), big + 5, 50_000_000, err.ptr)
    bs.wait_signal(flag.data_ptr(), big, 50_000_000, err.ptr)       # older target: done
    torch.cuda.synchronize()
    assert not err.set()
    bs.wait_signal(flag.data_ptr(), big + 6, 2_000_000, err.ptr)    # not reached: times out
    torch.cuda.synchronize()
    assert err.set()
    with pytest.raises(RuntimeError):
        err.check()


def test_epoch_signals_computed_on_device(bs):
    """bs_signals_epoch / bs_wait_signals_epoch: value = (*epoch) * mul + add on the device;
    bs_epoch_advance; captured in a CUDA graph, each replay uses the then-current epoch."""
    from paper_2510_13223_b200.transport import ErrorFlag
    ep = torch.full((1,), 2 ** 31 - 2, dtype=torch.int32, device="cuda")
    flags = torch.zeros(3, dtype=torch.int32, device="cuda")
    err = ErrorFlag()
    ptrs = [flags.data_ptr() + 4 * i for i in range(3)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        bs.epoch_advance(ep.data_ptr())            # 2^31 - 1
        bs.signals_epoch(ptrs, ep.data_ptr(), [1, 3, 1], [0, -2, 7])
        bs.wait_signals_epoch(ptrs, ep.data_ptr(), [1, 3, 1], [0, -2, 7], 50_000_000, err.ptr)
    torch.cuda.synchronize()
    e = 2 ** 31 - 1
    assert flags.cpu().tolist() == [bs.wrap_i32(e), bs.wrap_i32(3 * e - 2), bs.wrap_i32(e + 7)]
    assert not err.set()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        bs.epoch_advance(ep.data_ptr())
        bs.signals_epoch(ptrs[:1], ep.data_ptr(), 2, 1)
        bs.wait_signals_epoch(ptrs[:1], ep.data_ptr(), 2, 1, 50_000_000, err.ptr)
    for k in range(1, 4):                            # the epoch wraps on the first replay
        g.replay()
        torch.cuda.synchronize()
        assert int(ep.item()) == bs.wrap_i32(e + k)
        assert int(flags[0].item()) == bs.wrap_i32(2 * (e + k) + 1)
    assert not err.set()
