"""NEXT row F1: the Global KV Cache Store's CPU tier and its three-stage layer-wise
pipeline (§4.2, Figs. 5-6, eqs. 12-17).

The store is a paged pool in page-locked host memory (``KVPool(host=True)``).  Its
fetch (HtoD) and store (DtoH) legs move whole chunks between the store and a device
pool, bit-exact, by one of three engines:
  * ``"staged"`` (default) -- gather -> PCIe -> scatter, the H2 pattern on the host tier:
                 the copy engines move the chunks between the store's runs of consecutive
                 ids and ONE contiguous device staging buffer (one cudaMemcpyAsync per store
                 run, i.e. one per layer for a contiguous store extent), and the device side
                 is a scatter / gather kernel (``bs_kv_scatter_layer`` / ``bs_kv_gather_layer``,
                 HBM-speed, microseconds of SM time) into the pool's scattered blocks;
  * ``"ce"``  -- the copy engines only: ``bs_kv_migrate_layer_ce`` (one cudaMemcpyAsync
                 per run of ids consecutive on BOTH sides -- a fragmented device pool makes
                 that one small copy per chunk);
  * ``"sm"``  -- the copy kernel through the pages' UVA mapping over PCIe (zero-copy,
                 8 CTAs -- the rest of the GPU keeps computing).
``ThreeStagePipeline`` overlaps, per layer i (Fig. 6):

    HtoD stream : fetch the prefix KV of layer i+1 (lookahead 1)
    compute     : [wait fetch(i)] compute(i)
    DtoH stream : [wait compute(i)] store the incremental KV of layer i

The paper's transfer model (eqs. 12-13) is in ``oracle``; ``transfer_model`` here
restates it for the bench's prediction column only.
"""
from __future__ import annotations

import torch

from . import KVPool, copy_ptr, kv_gather_layer, kv_migrate_layer, kv_migrate_layer_ce, kv_scatter_layer


def _runs(ids):
    """[(first id, count, position)] of the runs of consecutive ids, in order."""
    out, i, ids = [], 0, [int(x) for x in ids]
    while i < len(ids):
        j = i + 1
        while j < len(ids) and ids[j] == ids[j - 1] + 1:
            j += 1
        out.append((ids[i], j - i, i))
        i = j
    return out


class StagedPairs:
    """A pair list prepared for the staged engine: the store side as runs of consecutive ids
    (host), the device side as a device int32 tensor, and a device staging buffer holding
    pair i's chunk at offset i * chunk_bytes.  The same pairs serve every layer; fetches and
    stores that may run concurrently need separate StagedPairs (separate staging)."""

    def __init__(self, store: "KVStore", dev: KVPool, store_ids, dev_ids):
        store_ids = [int(x) for x in store_ids]
        dev_ids = [int(x) for x in dev_ids]
        if len(store_ids) != len(dev_ids):
            raise ValueError("store_ids / dev_ids lengths differ")
        self.n = len(store_ids)
        self.runs = _runs(store_ids)
        self.dev_ids = torch.tensor(dev_ids, dtype=torch.int32, device=dev.device)
        self.staging = torch.empty(max(self.n, 1) * dev.chunk_bytes, dtype=torch.uint8,
                                   device=dev.device)


class KVStore:
    """CPU tier of the Global KV Cache Store: a pinned paged pool + its allocator."""

    def __init__(self, num_layers: int, num_blocks: int, num_kv_heads: int, head_dim: int):
        self.pool = KVPool(num_layers, num_blocks, num_kv_heads, head_dim, host=True)

    def alloc(self, n: int) -> list:
        return self.pool.alloc(n)

    def free(self, ids) -> None:
        self.pool.free(ids)

    def fetch_layer(self, dev: KVPool, layer: int, store_ids, dev_ids, stream=None,
                    engine: str = "sm") -> None:
        """HtoD: dev.chunk(layer, dev_ids[i]) <- store.chunk(layer, store_ids[i]).
        engine "sm": device int32 id tensors; "ce": host id lists."""
        if engine == "ce":
            kv_migrate_layer_ce(self.pool, dev, layer, store_ids, dev_ids, stream=stream)
        else:
            kv_migrate_layer(self.pool, dev, layer, store_ids, dev_ids, stream=stream)

    def store_layer(self, dev: KVPool, layer: int, dev_ids, store_ids, stream=None,
                    engine: str = "sm") -> None:
        """DtoH: store.chunk(layer, store_ids[i]) <- dev.chunk(layer, dev_ids[i])."""
        if engine == "ce":
            kv_migrate_layer_ce(dev, self.pool, layer, dev_ids, store_ids, stream=stream)
        else:
            kv_migrate_layer(dev, self.pool, layer, dev_ids, store_ids, stream=stream)


    # ---- staged engine ------------------------------------------------------------------
    def prepare(self, dev: KVPool, store_ids, dev_ids) -> StagedPairs:
        return StagedPairs(self, dev, store_ids, dev_ids)

    def _store_addr(self, layer: int, block: int) -> int:
        p = self.pool
        return p.data.data_ptr() + (layer * p.num_blocks + block) * p.chunk_bytes

    def fetch_staged(self, dev: KVPool, layer: int, sp: StagedPairs, stream=None) -> None:
        """HtoD: store runs -> staging (copy engines), staging -> dev blocks (scatter)."""
        if sp.n == 0:
            return
        cb = dev.chunk_bytes
        for first, cnt, pos in sp.runs:
            copy_ptr(sp.staging.data_ptr() + pos * cb, self._store_addr(layer, first), cnt * cb,
                     stream=stream)
        kv_scatter_layer(dev, layer, sp.dev_ids, sp.staging, stream=stream)

    def store_staged(self, dev: KVPool, layer: int, sp: StagedPairs, stream=None) -> None:
        """DtoH: dev blocks -> staging (gather), staging -> store runs (copy engines)."""
        if sp.n == 0:
            return
        cb = dev.chunk_bytes
        kv_gather_layer(dev, layer, sp.dev_ids, sp.staging, stream=stream)
        for first, cnt, pos in sp.runs:
            copy_ptr(self._store_addr(layer, first), sp.staging.data_ptr() + pos * cb, cnt * cb,
                     stream=stream)


def transfer_model(s_kv_bytes: float, l_tokens: float, r: float, bytes_per_s: float,
                   t_f_s: float, n_layers: int):
    """eqs. 12-13: T_F,layer = T_F r / N, T_KV = S_kv L r / B."""
    return t_f_s * r / n_layers, s_kv_bytes * l_tokens * r / bytes_per_s


class ThreeStagePipeline:
    def __init__(self, store: KVStore, dev: KVPool, num_layers: int, compute,
                 fetch_pairs=None, store_pairs=None, lookahead: int = 1, device=None,
                 engine: str = "staged"):
        """compute(layer) enqueues layer ``layer``'s work on the current stream.
        fetch_pairs = (store_ids, dev_ids), store_pairs = (dev_ids, store_ids): device
        int32 tensors (engine "sm") or host lists (engines "staged", "ce"), the same pairs
        every layer (block ids are shared by all layers)."""
        self.engine = engine
        self.store, self.dev, self.L = store, dev, num_layers
        if engine == "staged":   # host id lists -> prepared pairs with their own staging
            if fetch_pairs is not None:
                fetch_pairs = (store.prepare(dev, *fetch_pairs),)
            if store_pairs is not None:
                store_pairs = (store.prepare(dev, store_pairs[1], store_pairs[0]),)
        self.compute_fn = compute
        self.fetch_pairs, self.store_pairs = fetch_pairs, store_pairs
        self.lookahead = lookahead
        dev_ = device if device is not None else dev.device
        self.h2d = torch.cuda.Stream(device=dev_, priority=-1)
        self.d2h = torch.cuda.Stream(device=dev_, priority=-1)
        self.compute = torch.cuda.Stream(device=dev_)
        self.fetched = [torch.cuda.Event() for _ in range(num_layers)]
        self.computed = [torch.cuda.Event() for _ in range(num_layers)]
        self.started = [torch.cuda.Event() for _ in range(num_layers)]

    def enqueue(self, timers=None) -> None:
        """One pass over all layers.  timers[l] = (fetch_s, fetch_e, comp_s, comp_e,
        store_s, store_e) timing events recorded on the launching streams."""
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(cur)
        for s in (self.h2d, self.d2h, self.compute):
            s.wait_event(start)
        for layer in range(self.L):
            with torch.cuda.stream(self.h2d):
                if layer - self.lookahead >= 0:
                    self.h2d.wait_event(self.started[layer - self.lookahead])
                if timers is not None:
                    timers[layer][0].record(self.h2d)
                if self.fetch_pairs is not None and self.engine == "staged":
                    self.store.fetch_staged(self.dev, layer, self.fetch_pairs[0], stream=self.h2d)
                elif self.fetch_pairs is not None:
                    self.store.fetch_layer(self.dev, layer, *self.fetch_pairs, stream=self.h2d,
                                           engine=self.engine)
                if timers is not None:
                    timers[layer][1].record(self.h2d)
                self.fetched[layer].record(self.h2d)
            with torch.cuda.stream(self.compute):
                self.started[layer].record(self.compute)
                self.compute.wait_event(self.fetched[layer])
                if timers is not None:
                    timers[layer][2].record(self.compute)
                self.compute_fn(layer)
                if timers is not None:
                    timers[layer][3].record(self.compute)
                self.computed[layer].record(self.compute)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.computed[layer])
                if timers is not None:
                    timers[layer][4].record(self.d2h)
                if self.store_pairs is not None and self.engine == "staged":
                    self.store.store_staged(self.dev, layer, self.store_pairs[0], stream=self.d2h)
                elif self.store_pairs is not None:
                    self.store.store_layer(self.dev, layer, *self.store_pairs, stream=self.d2h,
                                           engine=self.engine)
                if timers is not None:
                    timers[layer][5].record(self.d2h)
        for s in (self.h2d, self.d2h, self.compute):
            cur.wait_stream(s)
