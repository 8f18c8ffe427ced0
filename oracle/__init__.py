"""fp64 CPU oracle for the BanaServe (arXiv 2510.13223) KV-migration + split-decode path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product package ``paper_2510_13223_b200`` never imports it, and this module never
imports the product package: the two share no code.

The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64, one OpenMP ``parallel
for`` over (request, head) rows in the attention loop, no SIMD intrinsics); this file
is argument marshalling over ctypes plus shape bookkeeping.  Each wrapper names the
PAPER.md passage its C function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f32 = ctypes.c_float
_f64 = ctypes.c_double
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (``-O2 -fopenmp``); returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.or_set_threads.argtypes = [_i32]
        L.or_set_threads.restype = None
        L.or_get_threads.argtypes = []
        L.or_get_threads.restype = _i32
        L.or_bf16_to_f64.argtypes = [ctypes.c_uint16]
        L.or_bf16_to_f64.restype = _f64
        L.or_kv_bytes_per_token_layer.argtypes = [_i32, _i32, _i32]
        L.or_kv_bytes_per_token_layer.restype = _i64
        L.or_kv_bytes_per_token.argtypes = [_i32, _i32, _i32, _i32]
        L.or_kv_bytes_per_token.restype = _i64
        L.or_t_f_layer_ms.argtypes = [_f64, _f64, _i32]
        L.or_t_f_layer_ms.restype = _f64
        L.or_t_kv_ms.argtypes = [_f64, _f64, _f64, _f64]
        L.or_t_kv_ms.restype = _f64
        L.or_layer_payload_bytes.argtypes = [_f64, _f64]
        L.or_layer_payload_bytes.restype = _f64
        L.or_t_layer_s.argtypes = [_f64, _f64, _f64]
        L.or_t_layer_s.restype = _f64
        L.or_chunk_elems.argtypes = [_i32, _i32, _i32]
        L.or_chunk_elems.restype = _i64
        L.or_pool_bytes.argtypes = [_i32, _i32, _i32, _i32, _i32]
        L.or_pool_bytes.restype = _i64
        L.or_pool_alloc.argtypes = [_p, _i32, _i32, _p]
        L.or_pool_alloc.restype = _i32
        L.or_pool_free.argtypes = [_p, _i32, _i32, _p]
        L.or_pool_free.restype = _i32
        L.or_migrate_layer.argtypes = [_p, _i32, _p, _i32, _i32, _i32, _i32, _i32, _p, _p, _i32]
        L.or_migrate_layer.restype = None
        L.or_migrate_heads_layer.argtypes = [_p, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32, _p,
                                             _p, _i32, _i32, _i32, _i32]
        L.or_migrate_heads_layer.restype = None
        L.or_append_token.argtypes = [_p, _i32, _i32, _i32, _i32, _i32, _p, _p, _i32, _p, _i32, _p]
        L.or_append_token.restype = None
        L.or_attention_shard.argtypes = [_p, _i32, _i32, _i32, _i32, _i32, _p, _i32, _i32, _p,
                                         _i32, _p, _i32, _i32, _f32, _p, _p, _p]
        L.or_attention_shard.restype = None
        L.or_merge_partials.argtypes = [_i32, _p, _p, _p, _i32, _i32, _i32, _p, _p]
        L.or_merge_partials.restype = None
        L.or_chained_two_shard.argtypes = [_p, _i32, _p, _i32, _p, _i32, _p, _i32, _i32, _i32,
                                           _i32, _i32, _p, _i32, _i32, _p, _f32, _p, _p]
        L.or_chained_two_shard.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


# --- eqs. 12-17 ---------------------------------------------------

def kv_bytes_per_token_layer(h_kv: int, d_head: int, elem_bytes: int = 2) -> int:
    """eq. 15."""
    return lib().or_kv_bytes_per_token_layer(h_kv, d_head, elem_bytes)


def kv_bytes_per_token(n_layers: int, h_kv: int, d_head: int, elem_bytes: int = 2) -> int:
    """eq. 16."""
    return lib().or_kv_bytes_per_token(n_layers, h_kv, d_head, elem_bytes)


def t_f_layer_ms(t_f_ms: float, r: float, n_layers: int) -> float:
    """eq. 12."""
    return lib().or_t_f_layer_ms(t_f_ms, r, n_layers)


def t_kv_ms(s_kv_bytes: float, l_tokens: float, r: float, b_gbps: float) -> float:
    """eq. 13, units per reading R-A17."""
    return lib().or_t_kv_ms(s_kv_bytes, l_tokens, r, b_gbps)


def layer_payload_bytes(s_w: float, s_kv: float) -> float:
    """eq. 3."""
    return lib().or_layer_payload_bytes(s_w, s_kv)


def t_layer_s(s_total: float, b_net: float, t_sync: float) -> float:
    """eq. 4; pinned to hand-worked layer sizes and closed forms
    (tests/golden/paper_eq3_4_hand.txt, tests/test_oracle_pins.py)."""
    return lib().or_t_layer_s(s_total, b_net, t_sync)


def migrate_layers(src_pool, dst_pool, layer_lo, n_layers, src_ids, dst_ids) -> None:
    """NEXT F3: migrate_layer for each layer of the range, in order."""
    for layer in range(layer_lo, layer_lo + n_layers):
        migrate_layer(src_pool, dst_pool, layer, src_ids, dst_ids)


# --- pool geometry and allocator (H0) ------------------------------------------------

def chunk_elems(h_kv: int, bs: int, d: int) -> int:
    return lib().or_chunk_elems(h_kv, bs, d)


def pool_bytes(n_layers: int, n_blocks: int, h_kv: int, bs: int, d: int) -> int:
    return lib().or_pool_bytes(n_layers, n_blocks, h_kv, bs, d)


class Allocator:
    """Lowest-free-id-first, all-or-nothing block allocator (reading R-A12)."""

    def __init__(self, n_blocks: int):
        self.used = np.zeros(n_blocks, dtype=np.uint8)

    def alloc(self, n: int) -> np.ndarray | None:
        out = np.zeros(max(n, 1), dtype=np.int32)
        rc = lib().or_pool_alloc(_ptr(self.used), len(self.used), n, _ptr(out))
        if rc == 2:
            return None
        if rc != 0:
            raise ValueError("invalid alloc")
        return out[:n].copy()

    def free(self, ids) -> bool:
        ids = _c(ids, np.int32)
        if ids.size == 0:
            ids = np.zeros(1, dtype=np.int32)[:0]
        buf = ids if ids.size else np.zeros(1, dtype=np.int32)
        return lib().or_pool_free(_ptr(self.used), len(self.used), int(ids.size), _ptr(buf)) == 0


# --- H2 migration --------------------------------------------------------------------

def migrate_layer(src_pool: np.ndarray, dst_pool: np.ndarray, layer: int, src_ids, dst_ids) -> None:
    """In-place on ``dst_pool`` (uint16 [L][NB][2][Hkv][bs][d])."""
    assert src_pool.dtype == np.uint16 and dst_pool.dtype == np.uint16
    L, nbs, two, hkv, bs, d = src_pool.shape
    assert dst_pool.shape[2:] == src_pool.shape[2:] and two == 2
    s = _c(src_ids, np.int32)
    t = _c(dst_ids, np.int32)
    assert s.shape == t.shape
    if s.size == 0:
        return
    lib().or_migrate_layer(_ptr(src_pool), nbs, _ptr(dst_pool), dst_pool.shape[1], hkv, bs, d,
                           layer, _ptr(s), _ptr(t), int(s.size))


def append_token(pool: np.ndarray, layer: int, k_new, v_new, block_tables, pos) -> None:
    """(H7) In place on ``pool`` (uint16 [L][NB][2][Hkv][bs][d]): the decoded token's K/V
    (uint16 bf16 bits [B][Hkv][d]) into local token ``pos[b]`` of each request's shard
    (block ``block_tables[b][pos // bs]``, slot ``pos % bs``); ``pos[b] < 0`` skips.
    The paper is silent (reading R-A9: the current token's K/V is in the cache)."""
    assert pool.dtype == np.uint16 and pool.flags.c_contiguous
    L, nb, two, hkv, bs, d = pool.shape
    k = _c(k_new, np.uint16)
    v = _c(v_new, np.uint16)
    bt = _c(block_tables, np.int32)
    p = _c(pos, np.int32)
    B = p.shape[0]
    assert k.shape == (B, hkv, d) and v.shape == (B, hkv, d) and bt.shape[0] == B
    if B == 0:
        return
    lib().or_append_token(_ptr(pool), nb, hkv, bs, d, layer, _ptr(k), _ptr(v), B, _ptr(bt),
                          bt.shape[1], _ptr(p))


def migrate_heads_layer(src_pool: np.ndarray, dst_pool: np.ndarray, layer: int, src_ids, dst_ids,
                        src_head_lo: int, dst_head_lo: int, n_heads: int) -> None:
    """NEXT F2: K/V pages of n_heads kv-heads, in place on dst_pool."""
    assert src_pool.dtype == np.uint16 and dst_pool.dtype == np.uint16
    _, nbs, _, shkv, bs, d = src_pool.shape
    _, nbd, _, dhkv, bs2, d2 = dst_pool.shape
    assert (bs, d) == (bs2, d2)
    assert 0 <= src_head_lo and src_head_lo + n_heads <= shkv
    assert 0 <= dst_head_lo and dst_head_lo + n_heads <= dhkv
    s = _c(src_ids, np.int32)
    t = _c(dst_ids, np.int32)
    if s.size == 0:
        return
    lib().or_migrate_heads_layer(_ptr(src_pool), nbs, shkv, _ptr(dst_pool), nbd, dhkv, bs, d, layer,
                                 _ptr(s), _ptr(t), int(s.size), src_head_lo, dst_head_lo, n_heads)


# --- H4 attention over one shard -------------------------------------------------------

def attention_shard(pool: np.ndarray, layer: int, q: np.ndarray, block_tables: np.ndarray,
                    kv_split: np.ndarray, shard_id: int, scale: float):
    """Returns (o [B,Hq,d] f64, m [B,Hq] f64, l [B,Hq] f64); eqs. 6-9.

    ``q`` is uint16 bf16 bits [B,Hq,d]; ``block_tables`` int32 [B,max_blocks];
    ``kv_split`` int32 [B, n_shards+1].
    """
    L, nb, two, hkv, bs, d = pool.shape
    q = _c(q, np.uint16)
    bt = _c(block_tables, np.int32)
    ks = _c(kv_split, np.int32)
    B, hq, dq = q.shape
    assert dq == d and hq % hkv == 0
    o = np.zeros((B, hq, d), dtype=np.float64)
    m = np.zeros((B, hq), dtype=np.float64)
    l = np.zeros((B, hq), dtype=np.float64)
    lib().or_attention_shard(_ptr(pool), nb, hkv, bs, d, layer, _ptr(q), B, hq, _ptr(bt),
                             bt.shape[1], _ptr(ks), ks.shape[1] - 1, shard_id,
                             np.float32(scale).item(), _ptr(o), _ptr(m), _ptr(l))
    return o, m, l


# --- H6 merge --------------------------------------------------------------------------

def merge_partials(o_parts, m_parts, l_parts):
    """Exact LSE merge (eq. 10, PAPER.md:233-235 + R-A4).  Returns (o f64, lse f64)."""
    o = _c(np.stack(o_parts), np.float64)
    m = _c(np.stack(m_parts), np.float64)
    l = _c(np.stack(l_parts), np.float64)
    n, B, hq, d = o.shape
    out = np.zeros((B, hq, d), dtype=np.float64)
    lse = np.zeros((B, hq), dtype=np.float64)
    lib().or_merge_partials(n, _ptr(o), _ptr(m), _ptr(l), B, hq, d, _ptr(out), _ptr(lse))
    return out, lse


def chained_two_shard(pool0, bt0, pool1, bt1, layer, q, kv_split, scale):
    """The paper's literal two-device protocol (eqs. 6-10, Fig. 4) with R-A3/R-A4."""
    L, nb0, _, hkv, bs, d = pool0.shape
    nb1 = pool1.shape[1]
    q = _c(q, np.uint16)
    b0 = _c(bt0, np.int32)
    b1 = _c(bt1, np.int32)
    ks = _c(kv_split, np.int32)
    assert ks.shape[1] == 3
    B, hq, _ = q.shape
    o = np.zeros((B, hq, d), dtype=np.float64)
    lse = np.zeros((B, hq), dtype=np.float64)
    lib().or_chained_two_shard(_ptr(pool0), nb0, _ptr(b0), b0.shape[1], _ptr(pool1), nb1,
                               _ptr(b1), b1.shape[1], hkv, bs, d, layer, _ptr(q), B, hq, _ptr(ks),
                               np.float32(scale).item(), _ptr(o), _ptr(lse))
    return o, lse


def attention_full(pools, block_tables, layer, q, kv_split, scale):
    """Convenience: all shards through ``attention_shard`` then ``merge_partials``."""
    parts = [attention_shard(p, layer, q, bt, kv_split, j, scale)
             for j, (p, bt) in enumerate(zip(pools, block_tables))]
    return merge_partials([x[0] for x in parts], [x[1] for x in parts], [x[2] for x in parts])


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (for timing reports: 1 thread vs all cores)."""
    lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(lib().or_get_threads())
