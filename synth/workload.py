"""Seeded synthetic workloads.

Value recipe (SURVEY.md §8(d) "Concrete synthetic inputs"):
  * q, k ~ N(0, 1); v ~ N(0, 1) + per-channel bias ~ U(-1, 1); rounded RNE to bf16
    (torch ``.to(bfloat16)``), reading R-A13.
  * per (layer, request, kv-head) ``n_needles`` needle keys at seeded positions:
    k = 10 * qbar / |qbar| with qbar the mean of the group's q heads, so a few scores
    sit ~10 above the bulk and cross-shard max rescaling is exercised.
  * pad slots of each shard's last block and every free block hold bf16 NaN 0x7FC0;
    destination pools are pre-filled with the sentinel 0xA5A5.
Lengths (Fig. 7): Alpaca-like U{5..40} prompts, LongBench-like
log-uniform[2000, 32768] (clipped from 85k), generated-so-far U{0..511}.

Layout of a pool: uint16 ``[L][num_blocks][2 (K,V)][Hkv][bs][d]`` (D4).
Randomness uses ``torch.Generator`` seeded per call, so values are identical on every
machine; everything is produced on the CPU unless a ``device`` is given.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

BF16_NAN = 0x7FC0
DST_SENTINEL = 0xA5A5
BLOCK_SIZE = 16


@dataclasses.dataclass(frozen=True)
class Shape:
    n_layers: int
    hq: int
    hkv: int
    d: int
    bs: int = BLOCK_SIZE

    @property
    def group(self) -> int:
        return self.hq // self.hkv

    @property
    def chunk_bytes(self) -> int:  # one (layer, block): K and V pages of all heads
        return 2 * self.hkv * self.bs * self.d * 2

    @property
    def kv_bytes_per_token_layer(self) -> int:
        return 2 * self.hkv * self.d * 2


# BASELINE.json "configs" (shapes only; batch/length recipes in make_* below).
TOY = Shape(n_layers=1, hq=4, hkv=2, d=64)
LLAMA2_7B = Shape(n_layers=32, hq=32, hkv=32, d=128)
LLAMA3_8B = Shape(n_layers=32, hq=32, hkv=8, d=128)
LLAMA2_70B = Shape(n_layers=80, hq=64, hkv=8, d=128)

TOY_SEQ_LENS = (37, 64, 129, 200)


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def bf16_bits(x: torch.Tensor) -> np.ndarray:
    """fp32 tensor -> numpy uint16 bf16 bit patterns (RNE via torch)."""
    return x.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


# ---------------------------------------------------------------------------------
# lengths and splits
# ---------------------------------------------------------------------------------

def mixed_lengths(n: int, seed: int, long_max: int = 32768) -> np.ndarray:
    """50% Alpaca-like U{5..40} prompts, 50% LongBench-like log-uniform[2000, long_max],
    plus generated-so-far U{0..511}."""
    g = _gen(seed)
    kind = torch.rand(n, generator=g) < 0.5
    short = torch.randint(5, 41, (n,), generator=g)
    lo, hi = math.log(2000.0), math.log(float(long_max))
    long_ = torch.exp(lo + (hi - lo) * torch.rand(n, generator=g)).floor().to(torch.int64)
    gen = torch.randint(0, 512, (n,), generator=g)
    lens = torch.where(kind, short, long_) + gen
    return lens.clamp(max=long_max).numpy().astype(np.int64)


def block_aligned_split(seq_lens, n_shards: int, bs: int = BLOCK_SIZE) -> np.ndarray:
    """kv_split [B, n+1]: shard j gets a contiguous, block-aligned token range; blocks
    are dealt as evenly as possible, earlier shards first; the last offset is seq_len
    (reading R-A11).  Short requests leave trailing shards empty."""
    lens = np.asarray(seq_lens, dtype=np.int64)
    out = np.zeros((len(lens), n_shards + 1), dtype=np.int32)
    for b, n in enumerate(lens):
        nblk = ceil_div(int(n), bs)
        per, extra = divmod(nblk, n_shards)
        off = 0
        for j in range(n_shards):
            off += (per + (1 if j < extra else 0)) * bs
            out[b, j + 1] = min(off, int(n))
    return out


def toy_split(seq_lens=TOY_SEQ_LENS, bs: int = BLOCK_SIZE) -> np.ndarray:
    """2-way split at 16*floor(len/32)."""
    lens = np.asarray(seq_lens, dtype=np.int64)
    s = (bs * (lens // (2 * bs))).astype(np.int32)
    return np.stack([np.zeros_like(s), s, lens.astype(np.int32)], axis=1)


def random_split(seq_lens, n_shards: int, seed: int) -> np.ndarray:
    """Arbitrary (unaligned, possibly empty) split points, for invariance tests."""
    g = _gen(seed)
    out = np.zeros((len(seq_lens), n_shards + 1), dtype=np.int32)
    for b, n in enumerate(seq_lens):
        cuts = torch.randint(0, int(n) + 1, (n_shards - 1,), generator=g).sort().values.numpy()
        out[b, 1:n_shards] = cuts
        out[b, n_shards] = n
    return out


# ---------------------------------------------------------------------------------
# dense values
# ---------------------------------------------------------------------------------

@dataclasses.dataclass
class DenseKV:
    """Per-request dense K/V bf16 bits: k[b] and v[b] are uint16 [L][len_b][Hkv][d];
    q is uint16 [L][B][Hq][d]."""
    shape: Shape
    seq_lens: np.ndarray
    q: np.ndarray
    k: list
    v: list


def gen_dense(shape: Shape, seq_lens, seed: int, n_needles: int = 4) -> DenseKV:
    g = _gen(seed)
    L, hq, hkv, d = shape.n_layers, shape.hq, shape.hkv, shape.d
    B = len(seq_lens)
    qf = torch.randn(L, B, hq, d, generator=g)
    q = bf16_bits(qf)
    qf = torch.from_numpy(q.view(np.int16)).view(torch.bfloat16).float()  # what the kernel sees
    bias = torch.rand(L, hkv, d, generator=g) * 2 - 1
    ks, vs = [], []
    for b, n in enumerate(seq_lens):
        n = int(n)
        kf = torch.randn(L, n, hkv, d, generator=g)
        vf = torch.randn(L, n, hkv, d, generator=g) + bias[:, None, :, :]
        if n > 0 and n_needles > 0:
            qbar = qf[:, b].reshape(L, hkv, shape.group, d).mean(dim=2)  # [L,Hkv,d]
            unit = qbar / qbar.norm(dim=-1, keepdim=True).clamp_min(1e-6)
            for layer in range(L):
                for kvh in range(hkv):
                    pos = torch.randint(0, n, (n_needles,), generator=g)
                    kf[layer, pos, kvh, :] = 10.0 * unit[layer, kvh]
        ks.append(bf16_bits(kf))
        vs.append(bf16_bits(vf))
    return DenseKV(shape, np.asarray(seq_lens, dtype=np.int64), q, ks, vs)


# ---------------------------------------------------------------------------------
# paged placement
# ---------------------------------------------------------------------------------

@dataclasses.dataclass
class ShardPool:
    pool: np.ndarray          # uint16 [L][NB][2][Hkv][bs][d]
    block_tables: np.ndarray  # int32 [B][max_blocks], -1 padded
    used: np.ndarray          # uint8 [NB], 1 where a block holds live tokens


def place_shards(dense: DenseKV, kv_split: np.ndarray, blocks_per_pool=None, seed: int = 0,
                 spare_blocks: int = 3, shuffle: bool = True) -> list:
    """Lay each shard's tokens into its own paged pool, shard-local order (token u of
    shard j at block bt[b][u//bs], slot u%bs).  Physical block ids come from a seeded
    permutation (a fragmented pool, as a serving engine leaves it).  Pad slots and free
    blocks are poisoned with bf16 NaN."""
    sh = dense.shape
    L, hkv, bs, d = sh.n_layers, sh.hkv, sh.bs, sh.d
    B = len(dense.seq_lens)
    n_shards = kv_split.shape[1] - 1
    g = _gen(seed + 7919)
    out = []
    for j in range(n_shards):
        lens = (kv_split[:, j + 1] - kv_split[:, j]).astype(np.int64)
        nblk = [ceil_div(int(x), bs) for x in lens]
        need = int(sum(nblk))
        nb = blocks_per_pool if blocks_per_pool is not None else need + spare_blocks
        assert nb >= need, "pool too small"
        perm = torch.randperm(nb, generator=g).numpy() if shuffle else np.arange(nb)
        pool = np.full((L, nb, 2, hkv, bs, d), BF16_NAN, dtype=np.uint16)
        mb = max(1, max(nblk) if nblk else 1)
        bt = np.full((B, mb), -1, dtype=np.int32)
        used = np.zeros(nb, dtype=np.uint8)
        nxt = 0
        for b in range(B):
            s0 = int(kv_split[b, j])
            for i in range(nblk[b]):
                blk = int(perm[nxt])
                nxt += 1
                bt[b, i] = blk
                used[blk] = 1
                lo = s0 + i * bs
                hi = min(s0 + lens[b], lo + bs)
                cnt = hi - lo
                # [L][cnt][Hkv][d] -> [L][Hkv][cnt][d]
                pool[:, blk, 0, :, :cnt, :] = dense.k[b][:, lo:hi].transpose(0, 2, 1, 3)
                pool[:, blk, 1, :, :cnt, :] = dense.v[b][:, lo:hi].transpose(0, 2, 1, 3)
        out.append(ShardPool(pool, bt, used))
    return out


def toy_case(seed: int = 0):
    """C1 toy: 1 layer, 4/2 heads, d=64, 4 requests {37,64,129,200}, 2-way split."""
    dense = gen_dense(TOY, TOY_SEQ_LENS, seed)
    ks = toy_split()
    return dense, ks, place_shards(dense, ks, seed=seed)


@dataclasses.dataclass
class DeviceShards:
    """Full-size case generated directly in device memory (bench / sampled parity).
    pools[j]: torch bf16 [L][NB][2][Hkv][bs][d]; block_tables[j]: numpy int32 [B][mb];
    kv_split numpy int32 [B][n+1]; q torch bf16 [L][B][Hq][d]."""
    shape: Shape
    seq_lens: np.ndarray
    kv_split: np.ndarray
    pools: list
    block_tables: list
    q: "torch.Tensor"


def device_pool(shape: Shape, shard_lens, seed: int, device, spare_blocks: int = 0,
                layers: int | None = None):
    """One paged pool holding one shard of every request (shard-local token order):
    seeded N(0,1) bf16 K, N(0,1) + per-channel bias V, generated on ``device`` with a torch
    generator; block placement from a seeded CPU permutation (a fragmented pool).  Pad
    slots keep random values (attention must mask them).  Returns (pool, block_table)."""
    L = shape.n_layers if layers is None else layers
    gd = torch.Generator(device=device)
    gd.manual_seed(int(seed))
    gc = _gen(int(seed) + 104729)
    lens = np.asarray(shard_lens, dtype=np.int64)
    B = len(lens)
    nblk = [ceil_div(int(x), shape.bs) for x in lens]
    nb = max(int(sum(nblk)) + spare_blocks, 1)
    perm = torch.randperm(nb, generator=gc).numpy()
    pool = torch.randn((L, nb, 2, shape.hkv, shape.bs, shape.d), generator=gd, device=device,
                       dtype=torch.bfloat16)
    bias = (torch.rand((L, shape.hkv, 1, shape.d), generator=gd, device=device) * 2 - 1)
    pool[:, :, 1] += bias.to(torch.bfloat16)[:, None]
    bt = np.full((B, max(1, max(nblk) if nblk else 1)), -1, dtype=np.int32)
    nxt = 0
    for b in range(B):
        bt[b, :nblk[b]] = perm[nxt:nxt + nblk[b]]
        nxt += nblk[b]
    return pool, bt


def device_q(shape: Shape, batch: int, seed: int, device, layers: int | None = None):
    L = shape.n_layers if layers is None else layers
    gd = torch.Generator(device=device)
    gd.manual_seed(int(seed) * 7919 + 17)
    return torch.randn((L, batch, shape.hq, shape.d), generator=gd, device=device,
                       dtype=torch.bfloat16)


def shard_seed(request_seed: int, shard: int) -> int:
    return int(request_seed) * 1000 + int(shard) + 1


def device_shards(shape: Shape, seq_lens, kv_split: np.ndarray, seed: int, device,
                  spare_blocks: int = 0, layers: int | None = None) -> DeviceShards:
    """Full-size case generated directly in device memory: one pool per shard
    (``device_pool`` with seed ``shard_seed(seed, j)``) and q (``device_q``)."""
    B = len(seq_lens)
    n = kv_split.shape[1] - 1
    pools, bts = [], []
    for j in range(n):
        lens = (kv_split[:, j + 1] - kv_split[:, j]).astype(np.int64)
        pool, bt = device_pool(shape, lens, shard_seed(seed, j), device, spare_blocks, layers)
        pools.append(pool)
        bts.append(bt)
    q = device_q(shape, B, seed, device, layers)
    return DeviceShards(shape, np.asarray(seq_lens), kv_split, pools, bts, q)


def extract_requests(case: DeviceShards, req_ids, layer: int):
    """Copy the blocks of a few requests of one layer to the host as a compact case
    (uint16 pools renumbered 0..k-1, block tables, kv_split, q) for the oracle."""
    req_ids = list(req_ids)
    pools, bts = [], []
    for pool, bt in zip(case.pools, case.block_tables):
        rows = bt[req_ids]
        ids = sorted({int(x) for x in rows.ravel() if x >= 0})
        remap = {x: i for i, x in enumerate(ids)}
        idx = torch.tensor(ids if ids else [0], dtype=torch.long, device=pool.device)
        sub = pool[layer:layer + 1].index_select(1, idx).cpu().view(torch.int16).numpy().view(np.uint16)
        nbt = np.vectorize(lambda x: remap.get(int(x), -1))(rows).astype(np.int32) if ids else rows
        pools.append(np.ascontiguousarray(sub))
        bts.append(np.ascontiguousarray(nbt))
    q = case.q[layer, req_ids].cpu().view(torch.int16).numpy().view(np.uint16)
    return pools, bts, np.ascontiguousarray(case.kv_split[req_ids]), np.ascontiguousarray(q)


def default_scale(d: int) -> float:
    """Reading R-A2: scale = 1/sqrt(d) rounded to fp32, passed to both sides."""
    return float(np.float32(1.0 / math.sqrt(d)))
