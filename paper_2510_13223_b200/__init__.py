"""B200-native (sm_100a) hot path of BanaServe (arXiv 2510.13223).

Thin ctypes binding over the C-ABI in ``include/banaserve.h`` (``libbanaserve.so``):
argument marshalling only -- every step of the path runs in the library's CUDA kernels.
PyTorch is used for device memory and streams.  There is no CPU fallback: importing
this package without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import build as _build

__all__ = [
    "BSError", "lib", "KVPool", "kv_migrate_layer", "kv_gather_layer", "kv_scatter_layer",
    "split_decode_attention", "split_decode_attention_workspace_size", "merge_partials",
    "MIGRATE_AUTO", "MIGRATE_VEC16", "MIGRATE_BULK", "EXPORTED_SYMBOLS",
]

ABI_VERSION = 2   # include/banaserve.h BS_ABI_VERSION this binding marshals for
MIGRATE_AUTO, MIGRATE_VEC16, MIGRATE_BULK = 0, 1, 2
BS_OK, BS_ERR_INVALID_ARG, BS_ERR_OUT_OF_BLOCKS, BS_ERR_UNSUPPORTED, BS_ERR_CUDA, BS_ERR_NCCL = range(6)

# every entry point include/banaserve.h declares
EXPORTED_SYMBOLS = (
    "bs_last_error", "bs_abi_version", "bs_kv_pool_bytes", "bs_kv_chunk_bytes",
    "bs_kv_pool_create", "bs_kv_pool_destroy", "bs_kv_pool_alloc", "bs_kv_pool_free",
    "bs_kv_pool_num_free", "bs_kv_migrate_layer", "bs_kv_migrate_layer_ex", "bs_kv_migrate_layer_ce",
    "bs_kv_gather_layer", "bs_kv_scatter_layer", "bs_split_decode_attention_workspace_size",
    "bs_split_decode_attention", "bs_merge_partials", "bs_nccl_unique_id_bytes",
    "bs_nccl_get_unique_id", "bs_comm_init", "bs_comm_destroy", "bs_sendrecv", "bs_kv_send_layer",
    "bs_kv_recv_layer", "bs_kv_sendrecv_layer", "bs_ipc_handle_bytes", "bs_ipc_export",
    "bs_ipc_import", "bs_ipc_close", "bs_kv_migrate_heads_layer",
    "bs_split_decode_attention_heads_workspace_size", "bs_split_decode_attention_heads",
    "bs_utilization", "bs_dispatch_requests", "bs_plan_migrations", "bs_kv_migrate_layers",
    "bs_copy_bytes", "bs_split_decode_attention_local_workspace_size",
    "bs_split_decode_attention_local", "bs_signal", "bs_wait_signal",
    "bs_attention_problem_workspace_size", "bs_split_decode_attention_tasks", "bs_wait_signals",
    "bs_signals", "bs_attention_ragged_plan", "bs_split_decode_attention_local_ragged",
    "bs_debug_build", "bs_debug_error_code", "bs_kv_append_token", "bs_exchange",
    "bs_signals_epoch", "bs_wait_signals_epoch", "bs_epoch_advance", "bs_kv_migrate_append_layer",
    "bs_split_decode_attention_local_ex", "bs_attention_last_launch",
    "bs_split_decode_attention_local_ragged_ex", "bs_attention_ragged_plan_ex",
)


class BSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[bs_status {status}] {msg}")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("num_layers", "num_blocks", "block_size", "num_kv_heads", "head_dim", "dtype",
                 "device")]


_i32, _p, _sz, _f32 = ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_float
_lib = None


def lib_path() -> str:
    """The library lib() loads: the debug build when BS_DEBUG=1."""
    if os.environ.get("BS_DEBUG") == "1":
        return _build.LIB_DEBUG
    return _build.LIB_TIMELINE if os.environ.get("BS_TIMELINE") == "1" else _build.LIB


def lib():
    """Load libbanaserve.so (building it if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    debug = os.environ.get("BS_DEBUG") == "1"   # device-side index checks (debug build)
    timeline = not debug and os.environ.get("BS_TIMELINE") == "1"  # kernel timeline stamps
    path = _build.LIB_DEBUG if debug else (_build.LIB_TIMELINE if timeline else _build.LIB)
    if os.environ.get("BS_LIB"):   # A/B experiments: another build of the library, as is
        path = os.environ["BS_LIB"]
    else:
        try:
            path = _build.build(debug=debug, timeline=timeline)
        except Exception as e:  # no nvcc on this machine: use the shipped .so if present
            if not os.path.exists(path):
                raise ImportError(f"libbanaserve.so missing and cannot be built: {e}") from e
    L = ctypes.CDLL(path)
    L.bs_abi_version.restype = ctypes.c_int32
    if L.bs_abi_version() != ABI_VERSION:   # the struct layouts below are this version's
        raise ImportError(f"{path}: ABI version {L.bs_abi_version()}, the binding needs "
                          f"{ABI_VERSION} -- rebuild (python -m paper_2510_13223_b200.build)")
    sig = {
        "bs_last_error": ([], ctypes.c_char_p),
        "bs_abi_version": ([], _i32),
        "bs_debug_build": ([], _i32),
        "bs_debug_error_code": ([_i32], _i32),
        "bs_attention_last_launch": ([_p, _p, _p, _p, _p], _i32),
        "bs_kv_pool_bytes": ([ctypes.POINTER(_Desc)], _sz),
        "bs_kv_chunk_bytes": ([ctypes.POINTER(_Desc)], _sz),
        "bs_kv_pool_create": ([ctypes.POINTER(_Desc), _p, ctypes.POINTER(_p)], _i32),
        "bs_kv_pool_destroy": ([_p], _i32),
        "bs_kv_pool_alloc": ([_p, _i32, _p], _i32),
        "bs_kv_pool_free": ([_p, _i32, _p], _i32),
        "bs_kv_pool_num_free": ([_p], _i32),
        "bs_kv_migrate_layer": ([_p, _p, _i32, _p, _p, _i32, _p], _i32),
        "bs_kv_migrate_layer_ex": ([_p, _p, _i32, _p, _p, _i32, _i32, _p], _i32),
        "bs_kv_migrate_layer_ce": ([_p, _p, _i32, _p, _p, _i32, _p], _i32),
        "bs_kv_append_token": ([_p, _i32, _p, _p, _i32, _p, _i32, _p, _p], _i32),
        "bs_kv_migrate_append_layer": ([_p, _p, _i32, _p, _p, _i32, _p, _p, _p, _i32, _p, _i32, _p,
                                        _p], _i32),
        "bs_kv_gather_layer": ([_p, _i32, _p, _i32, _p, _p], _i32),
        "bs_kv_scatter_layer": ([_p, _i32, _p, _i32, _p, _p], _i32),
        "bs_split_decode_attention_workspace_size": ([_p, _i32, _i32, _i32, ctypes.POINTER(_sz)], _i32),
        "bs_split_decode_attention": ([_p, _i32, _p, _i32, _i32, _p, _i32, _p, _i32, _i32, _f32,
                                       _p, _p, _p, _p, _sz, _p], _i32),
        "bs_merge_partials": ([_i32, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p], _i32),
        "bs_nccl_unique_id_bytes": ([], _sz),
        "bs_nccl_get_unique_id": ([_p], _i32),
        "bs_comm_init": ([_p, _i32, _i32, ctypes.POINTER(_p)], _i32),
        "bs_comm_destroy": ([_p], _i32),
        "bs_sendrecv": ([_p, _p, _sz, _i32, _p, _sz, _i32, _p], _i32),
        "bs_kv_send_layer": ([_p, _i32, _p, _i32, _i32, _p, _p, _p], _i32),
        "bs_kv_recv_layer": ([_p, _i32, _p, _i32, _i32, _p, _p, _p], _i32),
        "bs_kv_sendrecv_layer": ([_p, _p, _p, _i32, _i32, _p, _p, _p, _i32, _i32, _p, _i32, _p], _i32),
        "bs_ipc_handle_bytes": ([], _sz),
        "bs_ipc_export": ([_p, _p, ctypes.POINTER(_sz)], _i32),
        "bs_ipc_import": ([_p, _sz, ctypes.POINTER(_p)], _i32),
        "bs_ipc_close": ([_p, _sz], _i32),
        "bs_kv_migrate_heads_layer": ([_p, _p, _i32, _p, _p, _i32, _i32, _i32, _i32, _p], _i32),
        "bs_split_decode_attention_heads_workspace_size": ([_p, _i32, _i32, _i32, _i32, _i32,
                                                            ctypes.POINTER(_sz)], _i32),
        "bs_split_decode_attention_heads": ([_p, _i32, _i32, _i32, _i32, _i32, _p, _i32, _i32, _p,
                                             _i32, _p, _i32, _i32, _f32, _p, _p, _p, _p, _sz, _p],
                                            _i32),
        "bs_utilization": ([ctypes.c_double] * 4, ctypes.c_double),
        "bs_kv_migrate_layers": ([_p, _p, _i32, _i32, _p, _p, _i32, _p], _i32),
        "bs_copy_bytes": ([_p, _p, _sz, _p], _i32),
        "bs_signal": ([_p, _i32, _p], _i32),
        "bs_wait_signal": ([_p, _i32, ctypes.c_uint64, _p, _p], _i32),
        "bs_wait_signals": ([_i32, _p, _p, ctypes.c_uint64, _p, _p], _i32),
        "bs_signals": ([_i32, _p, _i32, _p], _i32),
        "bs_signals_epoch": ([_i32, _p, _p, _p, _p, _p], _i32),
        "bs_wait_signals_epoch": ([_i32, _p, _p, _p, _p, ctypes.c_uint64, _p, _p], _i32),
        "bs_epoch_advance": ([_p, _p], _i32),
        "bs_exchange": ([_p, _i32, _p, _p, _p, _i32, _p, _p, _p, _p], _i32),
        "bs_attention_ragged_plan": ([_i32, _i32, _p, _i32, _p, _i32, _i32, _i32, _i32, _p, _i32,
                                      ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                      ctypes.POINTER(_sz)], _i32),
        "bs_attention_ragged_plan_ex": ([_i32, _i32, _p, _i32, _p, _i32, _i32, _i32, _i32,
                                         ctypes.c_uint32, _p, _i32, ctypes.POINTER(_i32),
                                         ctypes.POINTER(_i32), ctypes.POINTER(_sz)], _i32),
        "bs_split_decode_attention_local_ragged": ([_i32, _p, _i32, _p, _i32, _i32, _p, _p, _p, _p,
                                                    _i32, _f32, _p, _i32, _i32, _p, _p, _p, _sz,
                                                    _p], _i32),
        "bs_split_decode_attention_local_ragged_ex": ([_i32, _p, _i32, _p, _i32, _i32, _p, _p, _p,
                                                       _p, _i32, _f32, _p, _i32, _i32, _p, _p, _p,
                                                       _sz, ctypes.c_uint32, _p], _i32),
        "bs_split_decode_attention_local_workspace_size": ([_i32, _p, _p, _i32, _i32,
                                                            ctypes.POINTER(_sz)], _i32),
        "bs_split_decode_attention_local": ([_i32, _p, _i32, _p, _i32, _i32, _p, _p, _p, _p, _i32,
                                             _f32, _p, _p, _p, _sz, _p], _i32),
        "bs_split_decode_attention_local_ex": ([_i32, _p, _i32, _p, _i32, _i32, _p, _p, _p, _p, _i32,
                                                _f32, _p, _p, _p, _sz, ctypes.c_uint32, _p], _i32),
        "bs_attention_problem_workspace_size": ([_i32, _i32, _i32, _i32, _i32, _p,
                                                 ctypes.POINTER(_sz)], _i32),
        "bs_split_decode_attention_tasks": ([_i32, _p, _i32, _p, _i32, _i32, _i32, _f32, _p], _i32),
        "bs_dispatch_requests": ([_i32, _p, _p, _i32, _p, ctypes.c_double, _p], _i32),
        "bs_plan_migrations": ([_i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, ctypes.c_double,
                                ctypes.c_double, _i32, _p, ctypes.POINTER(_i32)], _i32),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("BS_LIB") and not hasattr(L, name):
            continue   # an older build under A/B: its missing entry points stay unbound
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status: int) -> None:
    if status != BS_OK:
        raise BSError(status, lib().bs_last_error().decode())


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _dptr(t: torch.Tensor | None, dtype=None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"expected {dtype}, got {t.dtype}")
    return t.data_ptr()


class KVPool:
    """A paged bf16 KV pool ``[L][num_blocks][2][Hkv][16][head_dim]`` on one GPU.

    The device memory is a torch tensor (``self.data``); the C handle owns only the
    geometry and the block allocator (lowest-free-first, all-or-nothing).
    """

    def __init__(self, num_layers: int, num_blocks: int, num_kv_heads: int, head_dim: int,
                 device=None, base: torch.Tensor | None = None, block_size: int = 16,
                 host: bool = False):
        """``host=True``: a Global KV Cache Store tier pool in page-locked host memory
        (PAPER.md:248-254); only migrate / gather / scatter touch it."""
        if host:
            device = torch.device("cpu")
            dev_index = -1
        else:
            device = torch.device(device if device is not None else "cuda")
            if device.index is None:
                device = torch.device("cuda", torch.cuda.current_device())
            dev_index = device.index
        self.desc = _Desc(num_layers, num_blocks, block_size, num_kv_heads, head_dim, 0, dev_index)
        nbytes = lib().bs_kv_pool_bytes(ctypes.byref(self.desc))
        if nbytes == 0:
            raise BSError(BS_ERR_UNSUPPORTED, "unsupported pool geometry")
        if base is None:
            base = (torch.empty(nbytes // 2, dtype=torch.bfloat16, pin_memory=True) if host else
                    torch.empty(nbytes // 2, dtype=torch.bfloat16, device=device))
        if base.numel() * base.element_size() < nbytes:
            raise ValueError("base tensor too small")
        if host and not base.is_pinned():
            raise ValueError("host pools need page-locked (pinned) memory")
        self.base = base
        self.host = host
        self.data = base.view(torch.bfloat16).reshape(-1)[: nbytes // 2].view(
            num_layers, num_blocks, 2, num_kv_heads, block_size, head_dim)
        h = _p()
        _check(lib().bs_kv_pool_create(ctypes.byref(self.desc), base.data_ptr() if host else _dptr(base),
                                       ctypes.byref(h)))
        self.handle = h
        self.num_layers, self.num_blocks = num_layers, num_blocks
        self.num_kv_heads, self.head_dim, self.block_size = num_kv_heads, head_dim, block_size
        self.device = device
        self.nbytes = nbytes
        self.chunk_bytes = lib().bs_kv_chunk_bytes(ctypes.byref(self.desc))

    def alloc(self, n: int) -> list:
        buf = (ctypes.c_int32 * max(n, 1))()
        _check(lib().bs_kv_pool_alloc(self.handle, n, buf))
        return list(buf[:n])

    def free(self, ids) -> None:
        ids = [int(x) for x in ids]
        buf = (ctypes.c_int32 * max(len(ids), 1))(*ids)
        _check(lib().bs_kv_pool_free(self.handle, len(ids), buf))

    @property
    def num_free(self) -> int:
        return lib().bs_kv_pool_num_free(self.handle)

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().bs_kv_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kv_migrate_layer(src: KVPool, dst: KVPool, layer: int, src_ids: torch.Tensor,
                     dst_ids: torch.Tensor, method: int = MIGRATE_AUTO, stream=None) -> None:
    """H2: dst.chunk(layer, dst_ids[i]) <- src.chunk(layer, src_ids[i]) (device int32 ids)."""
    n = src_ids.numel()
    if dst_ids.numel() != n:
        raise ValueError("src_ids / dst_ids length mismatch")
    _check(lib().bs_kv_migrate_layer_ex(src.handle, dst.handle, layer,
                                        _dptr(src_ids, torch.int32), _dptr(dst_ids, torch.int32),
                                        n, method, _stream(stream)))


def kv_migrate_layer_ce(src: KVPool, dst: KVPool, layer: int, src_ids, dst_ids, stream=None) -> None:
    """H2 on the copy engines (DMA): host id lists; for the host-tier fetch / store legs."""
    s = [int(x) for x in src_ids]
    d = [int(x) for x in dst_ids]
    if len(s) != len(d):
        raise ValueError("src_ids / dst_ids length mismatch")
    n = len(s)
    sa = (ctypes.c_int32 * max(n, 1))(*s)
    da = (ctypes.c_int32 * max(n, 1))(*d)
    _check(lib().bs_kv_migrate_layer_ce(src.handle, dst.handle, layer, sa, da, n, _stream(stream)))


def kv_append_token(pool: KVPool, layer: int, k_new: torch.Tensor, v_new: torch.Tensor,
                    block_tables: torch.Tensor, pos: torch.Tensor, stream=None) -> None:
    """H7: the decoded token's K/V (bf16 [B, Hkv, d]) into local token ``pos[b]`` of each
    request's shard (device int32 ``pos``; < 0 skips)."""
    B = pos.numel()
    for t in (k_new, v_new):
        if t.dtype != torch.bfloat16 or not t.is_contiguous() or t.numel() != B * pool.num_kv_heads * pool.head_dim:
            raise ValueError("k_new / v_new must be contiguous bf16 [B, Hkv, d]")
    _check(lib().bs_kv_append_token(pool.handle, layer, _dptr(k_new, torch.bfloat16),
                                    _dptr(v_new, torch.bfloat16), B,
                                    _dptr(block_tables, torch.int32), int(block_tables.shape[1]),
                                    _dptr(pos, torch.int32), _stream(stream)))


def kv_migrate_append_layer(src: KVPool, dst: KVPool, layer: int, src_ids: torch.Tensor,
                            dst_ids: torch.Tensor, app_pool: KVPool, k_new: torch.Tensor,
                            v_new: torch.Tensor, block_tables: torch.Tensor, pos: torch.Tensor,
                            stream=None) -> None:
    """H2 + H7 in one launch: the hand-off copy src -> dst (device int32 ids) and the
    decoded token's K/V append into ``app_pool`` (see kv_append_token)."""
    n, B = src_ids.numel(), pos.numel()
    if dst_ids.numel() != n:
        raise ValueError("src_ids / dst_ids length mismatch")
    for t in (k_new, v_new):
        if (t.dtype != torch.bfloat16 or not t.is_contiguous()
                or t.numel() != B * app_pool.num_kv_heads * app_pool.head_dim):
            raise ValueError("k_new / v_new must be contiguous bf16 [B, Hkv, d]")
    _check(lib().bs_kv_migrate_append_layer(
        src.handle, dst.handle, layer, _dptr(src_ids, torch.int32), _dptr(dst_ids, torch.int32), n,
        app_pool.handle, _dptr(k_new, torch.bfloat16), _dptr(v_new, torch.bfloat16), B,
        _dptr(block_tables, torch.int32), int(block_tables.shape[1]), _dptr(pos, torch.int32),
        _stream(stream)))


def kv_gather_layer(src: KVPool, layer: int, ids: torch.Tensor, staging: torch.Tensor,
                    stream=None) -> None:
    _check(lib().bs_kv_gather_layer(src.handle, layer, _dptr(ids, torch.int32), ids.numel(),
                                    _dptr(staging), _stream(stream)))


def kv_scatter_layer(dst: KVPool, layer: int, ids: torch.Tensor, staging: torch.Tensor,
                     stream=None) -> None:
    _check(lib().bs_kv_scatter_layer(dst.handle, layer, _dptr(ids, torch.int32), ids.numel(),
                                     _dptr(staging), _stream(stream)))


def split_decode_attention_workspace_size(pool: KVPool, batch: int, num_q_heads: int,
                                          max_blocks: int) -> int:
    out = _sz()
    _check(lib().bs_split_decode_attention_workspace_size(pool.handle, batch, num_q_heads,
                                                          max_blocks, ctypes.byref(out)))
    return out.value


def split_decode_attention(pool: KVPool, layer: int, q: torch.Tensor, block_tables: torch.Tensor,
                           kv_split: torch.Tensor, shard_id: int, scale: float, o: torch.Tensor,
                           m: torch.Tensor, l: torch.Tensor, workspace: torch.Tensor | None = None,
                           stream=None) -> None:
    """H4: partial (o~, m, l) of shard ``shard_id`` for every request.

    q bf16 [B,Hq,d]; block_tables int32 [B,max_blocks]; kv_split int32 [B,n+1];
    o fp32 [B,Hq,d]; m, l fp32 [B,Hq]; workspace zero-filled once (see header)."""
    B, hq, d = q.shape
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().bs_split_decode_attention(
        pool.handle, layer, _dptr(q, torch.bfloat16), B, hq, _dptr(block_tables, torch.int32),
        block_tables.shape[1], _dptr(kv_split, torch.int32), kv_split.shape[1] - 1, shard_id,
        float(scale), _dptr(o, torch.float32), _dptr(m, torch.float32), _dptr(l, torch.float32),
        _dptr(workspace), ws_bytes, _stream(stream)))


def attention_last_launch() -> dict:
    """What this thread's most recent attention launch ran (bs_attention_last_launch):
    grid.x ranges, merge kind (MERGE_*; ``cluster`` = 1 for the cluster merge), programmatic
    dependent launch, tensor-core kernel, K/V stages per warp."""
    v = [ctypes.c_int32() for _ in range(5)]
    _check(lib().bs_attention_last_launch(*[ctypes.byref(x) for x in v]))
    r = dict(zip(("ranges", "merge", "pdl", "tensor_cores", "stages"), (int(x.value) for x in v)))
    r["cluster"] = int(r["merge"] == MERGE_CLUSTER)
    return r


def split_decode_attention_local_workspace_size(pools, max_blocks, batch: int,
                                                num_q_heads: int) -> int:
    n = len(pools)
    pa = (ctypes.c_void_p * n)(*[p.handle.value for p in pools])
    mb = (ctypes.c_int32 * n)(*[int(x) for x in max_blocks])
    out = _sz()
    _check(lib().bs_split_decode_attention_local_workspace_size(n, pa, mb, batch, num_q_heads,
                                                                ctypes.byref(out)))
    return out.value


ATTN_PDL = 1   # bs_split_decode_attention_local_ex flags (see the header's contract)
ATTN_NO_CLUSTER = 2
MERGE_NONE, MERGE_LAST_ARRIVER, MERGE_CLUSTER = 0, 1, 2   # attention_last_launch()["merge"]


def split_decode_attention_local(pools, layer: int, q: torch.Tensor, block_tables,
                                 shard_ids, kv_split: torch.Tensor, scale: float, out: torch.Tensor,
                                 lse: torch.Tensor, workspace: torch.Tensor | None = None,
                                 stream=None, flags: int = 0) -> None:
    """H4+H6 fused over shards resident on this GPU: bf16 ``out`` [B,Hq,d] + fp32 ``lse``.
    ``flags``: ATTN_PDL (programmatic dependent launch), ATTN_NO_CLUSTER (workspace merge
    instead of the cluster merge) -- bs_split_decode_attention_local_ex."""
    n = len(pools)
    B, hq, d = q.shape
    pa = (ctypes.c_void_p * n)(*[p.handle.value for p in pools])
    ba = (ctypes.c_void_p * n)(*[_dptr(t, torch.int32) for t in block_tables])
    mb = (ctypes.c_int32 * n)(*[int(t.shape[1]) for t in block_tables])
    sa = (ctypes.c_int32 * n)(*[int(x) for x in shard_ids])
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().bs_split_decode_attention_local_ex(
        n, pa, layer, _dptr(q, torch.bfloat16), B, hq, ba, mb, sa, _dptr(kv_split, torch.int32),
        kv_split.shape[1] - 1, float(scale), _dptr(out, torch.bfloat16),
        _dptr(lse, torch.float32) if lse is not None else None, _dptr(workspace), ws_bytes,
        int(flags), _stream(stream)))


class _Problem(ctypes.Structure):
    _fields_ = [("q", _p), ("kv_split", _p), ("n_shards", _i32), ("max_blocks", _p),
                ("out", _p), ("lse", _p), ("workspace", _p), ("workspace_bytes", _sz),
                ("done", _p), ("cross_device", _i32)]


class _Task(ctypes.Structure):
    _fields_ = [("pool", _p), ("block_tables", _p), ("shard_id", _i32), ("problem", _i32),
                ("order", _p)]


def _aptr(x, dtype=None):
    """Device pointer of a tensor, or an int address as is (e.g. a peer mapping)."""
    if x is None or isinstance(x, int):
        return x
    return _dptr(x, dtype)


def attention_problem_workspace_size(batch: int, num_q_heads: int, num_kv_heads: int,
                                     head_dim: int, max_blocks) -> int:
    n = len(max_blocks)
    mb = (ctypes.c_int32 * n)(*[int(x) for x in max_blocks])
    out = _sz()
    _check(lib().bs_attention_problem_workspace_size(batch, num_q_heads, num_kv_heads, head_dim, n,
                                                     mb, ctypes.byref(out)))
    return out.value


def split_decode_attention_tasks(problems, tasks, layer: int, batch: int, num_q_heads: int,
                                 scale: float, stream=None) -> None:
    """H4+H5+H6 fused across launches / GPUs (bs_split_decode_attention_tasks).
    ``problems``: dicts with q, kv_split, max_blocks (list), out, lse, workspace,
    workspace_bytes, done, cross_device -- tensors, or int addresses for peer mappings.
    ``tasks``: (pool, block_tables, shard_id, problem index[, order]) tuples -- ``order``: a
    device int32 permutation of the requests (dispatch order, e.g. longest first) or None."""
    keep = []
    pa = (_Problem * len(problems))()
    for i, pr in enumerate(problems):
        mb = (ctypes.c_int32 * len(pr["max_blocks"]))(*[int(x) for x in pr["max_blocks"]])
        keep.append(mb)
        ws = pr.get("workspace")
        wsb = pr.get("workspace_bytes")
        if wsb is None:
            wsb = 0 if ws is None or isinstance(ws, int) else ws.numel() * ws.element_size()
        pa[i] = _Problem(_aptr(pr["q"], torch.bfloat16), _aptr(pr["kv_split"], torch.int32),
                         len(pr["max_blocks"]), ctypes.cast(mb, _p), _aptr(pr["out"], torch.bfloat16),
                         _aptr(pr.get("lse"), torch.float32), _aptr(ws), wsb,
                         _aptr(pr.get("done"), torch.int32), int(bool(pr.get("cross_device", False))))
    ta = (_Task * len(tasks))()
    for t, task in enumerate(tasks):
        pool, bt, shard, prob = task[:4]
        order = task[4] if len(task) > 4 else None
        ta[t] = _Task(pool.handle.value, _dptr(bt, torch.int32), int(shard), int(prob),
                      _dptr(order, torch.int32) if order is not None else None)
    _check(lib().bs_split_decode_attention_tasks(len(problems), pa, len(tasks), ta, layer, batch,
                                                 num_q_heads, float(scale), _stream(stream)))


class RaggedPlan:
    """Host result of bs_attention_ragged_plan: ``work`` int32 [n][4] (copy to the device
    with :meth:`to`), ``max_parts`` and ``workspace_bytes``."""

    def __init__(self, work, max_parts, workspace_bytes):
        self.work, self.max_parts, self.workspace_bytes = work, max_parts, workspace_bytes
        self.n_work = int(work.shape[0])
        self.device_work = None

    def to(self, device):
        self.device_work = torch.from_numpy(self.work).to(device)
        return self


PLAN_PACK_SHORT = 1   # bs_attention_ragged_plan_ex flag


def attention_ragged_plan(kv_split_host, shard_ids, num_q_heads: int, num_kv_heads: int,
                          head_dim: int, max_blocks_per_range: int = 0,
                          pack_short: bool = False) -> RaggedPlan:
    """Host ragged plan (bs_attention_ragged_plan_ex).  ``pack_short``: requests of at most
    8 blocks in the (single) local shard are packed four to a CTA, one warp each."""
    import numpy as np
    ks = np.ascontiguousarray(np.asarray(kv_split_host, dtype=np.int32))
    B, n1 = ks.shape
    n = len(shard_ids)
    sa = (ctypes.c_int32 * n)(*[int(x) for x in shard_ids])
    nw, mp, wsb = _i32(), _i32(), _sz()
    args = (B, n1 - 1, ks.ctypes.data, n, sa, num_q_heads, num_kv_heads, head_dim,
            max_blocks_per_range, PLAN_PACK_SHORT if pack_short else 0)
    _check(lib().bs_attention_ragged_plan_ex(*args, None, 0, ctypes.byref(nw), ctypes.byref(mp),
                                             ctypes.byref(wsb)))
    work = np.zeros((nw.value, 4), dtype=np.int32)
    _check(lib().bs_attention_ragged_plan_ex(*args, work.ctypes.data, nw.value, ctypes.byref(nw),
                                             ctypes.byref(mp), ctypes.byref(wsb)))
    return RaggedPlan(work, mp.value, wsb.value)


def split_decode_attention_local_ragged(pools, layer: int, q: torch.Tensor, block_tables,
                                        shard_ids, kv_split: torch.Tensor, scale: float,
                                        plan: RaggedPlan, out: torch.Tensor, lse: torch.Tensor,
                                        workspace: torch.Tensor | None = None, stream=None,
                                        flags: int = 0) -> None:
    """H4+H6 fused over local shards, CTAs from a ragged plan (``plan.to(device)`` first).
    ``flags``: ATTN_PDL (bs_split_decode_attention_local_ragged_ex)."""
    n = len(pools)
    B, hq, d = q.shape
    pa = (ctypes.c_void_p * n)(*[p.handle.value for p in pools])
    ba = (ctypes.c_void_p * n)(*[_dptr(t, torch.int32) for t in block_tables])
    mb = (ctypes.c_int32 * n)(*[int(t.shape[1]) for t in block_tables])
    sa = (ctypes.c_int32 * n)(*[int(x) for x in shard_ids])
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().bs_split_decode_attention_local_ragged_ex(
        n, pa, layer, _dptr(q, torch.bfloat16), B, hq, ba, mb, sa, _dptr(kv_split, torch.int32),
        kv_split.shape[1] - 1, float(scale), _dptr(plan.device_work, torch.int32), plan.n_work,
        plan.max_parts, _dptr(out, torch.bfloat16),
        _dptr(lse, torch.float32) if lse is not None else None, _dptr(workspace), ws_bytes,
        int(flags), _stream(stream)))


def merge_partials(o_parts, m_parts, l_parts, out: torch.Tensor, lse: torch.Tensor | None = None,
                   stream=None) -> None:
    """H6: exact LSE merge of n partials into bf16 ``out`` [B,Hq,d] (+ fp32 lse [B,Hq])."""
    n = len(o_parts)
    B, hq, d = out.shape
    arr = ctypes.c_void_p * n
    o_arr = arr(*[_dptr(t, torch.float32) for t in o_parts])
    m_arr = arr(*[_dptr(t, torch.float32) for t in m_parts])
    l_arr = arr(*[_dptr(t, torch.float32) for t in l_parts])
    _check(lib().bs_merge_partials(n, o_arr, m_arr, l_arr, B, hq, d, _dptr(out, torch.bfloat16),
                                   _dptr(lse, torch.float32) if lse is not None else None,
                                   _stream(stream)))


# ---------------------------------------------------------------------------------------
# transports: NCCL (two-sided) and CUDA IPC (peer-mapped remote views for P2P push)
# ---------------------------------------------------------------------------------------

class Comm:
    """NCCL communicator owned by the library (``bs_comm``).  ``unique_id`` (bytes) is
    created by rank 0 with :func:`nccl_unique_id` and broadcast by the harness."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        h = _p()
        buf = ctypes.create_string_buffer(unique_id, len(unique_id))
        _check(lib().bs_comm_init(buf, nranks, rank, ctypes.byref(h)))
        self.handle, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if getattr(self, "handle", None):
            lib().bs_comm_destroy(self.handle)
            self.handle = None

    def sendrecv(self, send: torch.Tensor | None, send_peer: int, recv: torch.Tensor | None,
                 recv_peer: int, stream=None) -> None:
        sb = 0 if send is None else send.numel() * send.element_size()
        rb = 0 if recv is None else recv.numel() * recv.element_size()
        _check(lib().bs_sendrecv(self.handle, _dptr(send), sb, send_peer if send is not None else -1,
                                 _dptr(recv), rb, recv_peer if recv is not None else -1,
                                 _stream(stream)))


    def exchange(self, sends, recvs, stream=None) -> None:
        """One NCCL group of raw-byte sends [(tensor, peer)] and receives [(tensor, peer)]
        (bs_exchange) on ``stream``."""
        ns, nr = len(sends), len(recvs)
        sb = (ctypes.c_void_p * max(ns, 1))(*[_dptr(t) for t, _ in sends])
        sz = (ctypes.c_size_t * max(ns, 1))(*[t.numel() * t.element_size() for t, _ in sends])
        sp = (ctypes.c_int32 * max(ns, 1))(*[int(p) for _, p in sends])
        rb = (ctypes.c_void_p * max(nr, 1))(*[_dptr(t) for t, _ in recvs])
        rz = (ctypes.c_size_t * max(nr, 1))(*[t.numel() * t.element_size() for t, _ in recvs])
        rp = (ctypes.c_int32 * max(nr, 1))(*[int(p) for _, p in recvs])
        _check(lib().bs_exchange(self.handle, ns, sb, sz, sp, nr, rb, rz, rp, _stream(stream)))


def nccl_unique_id() -> bytes:
    n = lib().bs_nccl_unique_id_bytes()
    buf = ctypes.create_string_buffer(n)
    _check(lib().bs_nccl_get_unique_id(buf))
    return buf.raw


def kv_send_layer(src: KVPool, layer: int, ids: torch.Tensor, peer: int, comm: Comm,
                  staging: torch.Tensor, stream=None) -> None:
    _check(lib().bs_kv_send_layer(src.handle, layer, _dptr(ids, torch.int32), ids.numel(), peer,
                                  comm.handle, _dptr(staging), _stream(stream)))


def kv_recv_layer(dst: KVPool, layer: int, ids: torch.Tensor, peer: int, comm: Comm,
                  staging: torch.Tensor, stream=None) -> None:
    _check(lib().bs_kv_recv_layer(dst.handle, layer, _dptr(ids, torch.int32), ids.numel(), peer,
                                  comm.handle, _dptr(staging), _stream(stream)))


def kv_sendrecv_layer(comm: Comm, src: KVPool, src_ids: torch.Tensor, send_peer: int,
                      send_staging: torch.Tensor, dst: KVPool, dst_ids: torch.Tensor,
                      recv_peer: int, recv_staging: torch.Tensor, layer: int, stream=None) -> None:
    _check(lib().bs_kv_sendrecv_layer(
        comm.handle, src.handle, _dptr(src_ids, torch.int32), src_ids.numel(), send_peer,
        _dptr(send_staging), dst.handle, _dptr(dst_ids, torch.int32), dst_ids.numel(), recv_peer,
        _dptr(recv_staging), layer, _stream(stream)))


def _expandable_segments() -> bool:
    conf = os.environ.get("PYTORCH_CUDA_ALLOC_CONF", "") + "," + os.environ.get("PYTORCH_ALLOC_CONF", "")
    return any(x.replace(" ", "").lower() == "expandable_segments:true" for x in conf.split(","))


def ipc_export(t: torch.Tensor):
    """(handle bytes, offset) naming ``t``'s device memory for another process.  Needs memory
    from cudaMalloc: torch's expandable segments (virtual-memory mappings) cannot be exported
    with cudaIpcGetMemHandle, so that allocator mode is refused up front."""
    if _expandable_segments():
        raise BSError(BS_ERR_UNSUPPORTED, "ipc_export: PYTORCH_CUDA_ALLOC_CONF has expandable_segments:True -- its "
                      "virtual-memory segments cannot be IPC-exported; the P2P transport needs the "
                      "default caching allocator (or use the NCCL transport)")
    n = lib().bs_ipc_handle_bytes()
    buf = ctypes.create_string_buffer(n)
    off = _sz()
    _check(lib().bs_ipc_export(_dptr(t), buf, ctypes.byref(off)))
    return buf.raw, off.value


def ipc_import(handle: bytes, offset: int) -> int:
    """Device address (int) of an exported allocation + offset, mapped in this process."""
    out = _p()
    buf = ctypes.create_string_buffer(handle, len(handle))
    _check(lib().bs_ipc_import(buf, offset, ctypes.byref(out)))
    return out.value


def ipc_close(ptr: int, offset: int) -> None:
    _check(lib().bs_ipc_close(ptr, offset))


# ---------------------------------------------------------------------------------------
# NEXT F2: head-granular migration + attention over a kv-head range
# ---------------------------------------------------------------------------------------

def kv_migrate_heads_layer(src: KVPool, dst: KVPool, layer: int, src_ids: torch.Tensor,
                           dst_ids: torch.Tensor, src_head_lo: int, dst_head_lo: int, n_heads: int,
                           stream=None) -> None:
    _check(lib().bs_kv_migrate_heads_layer(src.handle, dst.handle, layer,
                                           _dptr(src_ids, torch.int32), _dptr(dst_ids, torch.int32),
                                           src_ids.numel(), src_head_lo, dst_head_lo, n_heads,
                                           _stream(stream)))


def split_decode_attention_heads_workspace_size(pool: KVPool, batch: int, n_kv_heads: int,
                                                num_kv_heads_total: int, num_q_heads: int,
                                                max_blocks: int) -> int:
    out = _sz()
    _check(lib().bs_split_decode_attention_heads_workspace_size(
        pool.handle, batch, n_kv_heads, num_kv_heads_total, num_q_heads, max_blocks, ctypes.byref(out)))
    return out.value


def split_decode_attention_heads(pool: KVPool, layer: int, pool_head_lo: int, model_head_lo: int,
                                 n_kv_heads: int, num_kv_heads_total: int, q: torch.Tensor,
                                 block_tables: torch.Tensor, kv_split: torch.Tensor, shard_id: int,
                                 scale: float, o: torch.Tensor, m: torch.Tensor, l: torch.Tensor,
                                 workspace: torch.Tensor | None = None, stream=None) -> None:
    B, hq, d = q.shape
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().bs_split_decode_attention_heads(
        pool.handle, layer, pool_head_lo, model_head_lo, n_kv_heads, num_kv_heads_total,
        _dptr(q, torch.bfloat16), B, hq, _dptr(block_tables, torch.int32), block_tables.shape[1],
        _dptr(kv_split, torch.int32), kv_split.shape[1] - 1, shard_id, float(scale),
        _dptr(o, torch.float32), _dptr(m, torch.float32), _dptr(l, torch.float32),
        _dptr(workspace), ws_bytes, _stream(stream)))


# ---------------------------------------------------------------------------------------
# NEXT F3: layer-level migration (KV of a contiguous layer range + weight tensors)
# ---------------------------------------------------------------------------------------

def kv_migrate_layers(src: KVPool, dst: KVPool, layer_lo: int, n_layers: int,
                      src_ids: torch.Tensor, dst_ids: torch.Tensor, stream=None) -> None:
    _check(lib().bs_kv_migrate_layers(src.handle, dst.handle, layer_lo, n_layers,
                                      _dptr(src_ids, torch.int32), _dptr(dst_ids, torch.int32),
                                      src_ids.numel(), _stream(stream)))


def copy_bytes(dst: torch.Tensor, src: torch.Tensor, stream=None) -> None:
    nb = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() < nb:
        raise ValueError("dst too small")
    _check(lib().bs_copy_bytes(dst.data_ptr(), src.data_ptr(), nb, _stream(stream)))


def migrate_layers(src: KVPool, dst: KVPool, layer_lo: int, n_layers: int, src_ids: torch.Tensor,
                   dst_ids: torch.Tensor, weights=(), stream=None) -> int:
    """Layer-level migration (Fig. 3): the KV of layers
    [layer_lo, layer_lo + n_layers) for the given block pairs plus each (src, dst) weight
    tensor pair W_l.  Returns the payload S_total = S_w + S_kv in bytes (eq. 3)."""
    kv_migrate_layers(src, dst, layer_lo, n_layers, src_ids, dst_ids, stream=stream)
    s_w = 0
    for ws, wd in weights:
        copy_bytes(wd, ws, stream=stream)
        s_w += ws.numel() * ws.element_size()
    return s_w + n_layers * src_ids.numel() * src.chunk_bytes


def t_layer_model(s_total_bytes: float, b_net_bytes_per_s: float, t_sync_s: float = 0.0) -> float:
    """eq. 4: T_layer ~= S_total / B_net + T_sync."""
    return s_total_bytes / b_net_bytes_per_s + t_sync_s


def wrap_i32(x: int) -> int:
    """x as the int32 the device holds (flags and counters wrap after 2^31; the waits
    compare wrap-safely)."""
    return ((int(x) + (1 << 31)) % (1 << 32)) - (1 << 31)


def signal(flag_ptr: int, value: int, stream=None) -> None:
    """After all prior work on the stream: *flag = value (flag may be peer-mapped)."""
    _check(lib().bs_signal(flag_ptr, wrap_i32(value), _stream(stream)))


def wait_signal(flag_ptr: int, value: int, timeout_ns: int = 0, err_ptr: int | None = None,
                stream=None) -> None:
    """The stream waits until *flag >= value, wrap-safe (gives up after timeout_ns,
    setting *err)."""
    _check(lib().bs_wait_signal(flag_ptr, wrap_i32(value), int(timeout_ns), err_ptr, _stream(stream)))


def signals(flag_ptrs, value: int, stream=None) -> None:
    """One launch: after all prior work on the stream, *flag_ptrs[i] = value (<= 16)."""
    n = len(flag_ptrs)
    fa = (ctypes.c_void_p * n)(*[int(f) for f in flag_ptrs])
    _check(lib().bs_signals(n, fa, wrap_i32(value), _stream(stream)))


def wait_signals(flag_ptrs, values, timeout_ns: int = 0, err_ptr: int | None = None,
                 stream=None) -> None:
    """One launch: the stream waits until *flag_ptrs[i] >= values[i] for every i (<= 16)."""
    n = len(flag_ptrs)
    fa = (ctypes.c_void_p * n)(*[int(f) for f in flag_ptrs])
    va = (ctypes.c_int32 * n)(*[wrap_i32(v) for v in values])
    _check(lib().bs_wait_signals(n, fa, va, int(timeout_ns), err_ptr, _stream(stream)))


def _epoch_arrays(flag_ptrs, mul, add):
    n = len(flag_ptrs)
    mul = [mul] * n if isinstance(mul, int) else list(mul)
    add = [add] * n if isinstance(add, int) else list(add)
    if len(mul) != n or len(add) != n:
        raise ValueError("flags / mul / add length mismatch")
    return (n, (ctypes.c_void_p * n)(*[int(f) for f in flag_ptrs]),
            (ctypes.c_int32 * n)(*[wrap_i32(v) for v in mul]),
            (ctypes.c_int32 * n)(*[wrap_i32(v) for v in add]))


def signals_epoch(flag_ptrs, epoch_ptr: int, mul=1, add=0, stream=None) -> None:
    """One launch: after all prior work on the stream, *flag_ptrs[i] = (*epoch) * mul[i] +
    add[i], computed on the device (CUDA-graph capturable steps)."""
    n, fa, ma, aa = _epoch_arrays(flag_ptrs, mul, add)
    _check(lib().bs_signals_epoch(n, fa, ma, aa, int(epoch_ptr), _stream(stream)))


def wait_signals_epoch(flag_ptrs, epoch_ptr: int, mul=1, add=0, timeout_ns: int = 0,
                       err_ptr: int | None = None, stream=None) -> None:
    """One launch: the stream waits until *flag_ptrs[i] >= (*epoch) * mul[i] + add[i]
    (device-computed, wrap-safe) for every i (<= 16)."""
    n, fa, ma, aa = _epoch_arrays(flag_ptrs, mul, add)
    _check(lib().bs_wait_signals_epoch(n, fa, ma, aa, int(epoch_ptr), int(timeout_ns), err_ptr,
                                       _stream(stream)))


def epoch_advance(epoch_ptr: int, stream=None) -> None:
    """Enqueue *epoch += 1 (the device step counter of a graph-capturable step)."""
    _check(lib().bs_epoch_advance(int(epoch_ptr), _stream(stream)))


def copy_ptr(dst_ptr: int, src_ptr: int, nbytes: int, stream=None) -> None:
    """Raw device / peer / host copy by address (copy engine)."""
    _check(lib().bs_copy_bytes(dst_ptr, src_ptr, nbytes, _stream(stream)))


def pool_view(num_layers: int, num_blocks: int, num_kv_heads: int, head_dim: int, ptr: int,
              device_index: int):
    """A pool handle over raw (e.g. peer-mapped) memory: the remote view a P2P push
    writes into.  Returns an object with ``.handle`` usable by the migrate calls."""
    desc = _Desc(num_layers, num_blocks, 16, num_kv_heads, head_dim, 0, device_index)
    h = _p()
    _check(lib().bs_kv_pool_create(ctypes.byref(desc), ptr, ctypes.byref(h)))

    class _View:
        pass
    v = _View()
    v.handle, v.desc = h, desc
    v.num_layers, v.num_blocks, v.num_kv_heads, v.head_dim = num_layers, num_blocks, num_kv_heads, head_dim
    v.chunk_bytes = lib().bs_kv_chunk_bytes(ctypes.byref(desc))
    return v
