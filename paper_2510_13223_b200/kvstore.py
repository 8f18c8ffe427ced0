"""NEXT row F1: the Global KV Cache Store's CPU tier and its three-stage layer-wise
pipeline (§4.2, Figs. 5-6, eqs. 12-17).

The store is a paged pool in page-locked host memory (``KVPool(host=True)``).  Its
fetch (HtoD) and store (DtoH) legs move whole chunks between the store and a device
pool, bit-exact, by one of two engines:
  * ``"ce"``  -- the copy engines: ``bs_kv_migrate_layer_ce`` (one cudaMemcpyAsync
                 per run of consecutive ids); no SM time at all;
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

from . import KVPool, kv_migrate_layer, kv_migrate_layer_ce


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


def transfer_model(s_kv_bytes: float, l_tokens: float, r: float, bytes_per_s: float,
                   t_f_s: float, n_layers: int):
    """eqs. 12-13: T_F,layer = T_F r / N, T_KV = S_kv L r / B."""
    return t_f_s * r / n_layers, s_kv_bytes * l_tokens * r / bytes_per_s


class ThreeStagePipeline:
    def __init__(self, store: KVStore, dev: KVPool, num_layers: int, compute,
                 fetch_pairs=None, store_pairs=None, lookahead: int = 1, device=None,
                 engine: str = "ce"):
        """compute(layer) enqueues layer ``layer``'s work on the current stream.
        fetch_pairs = (store_ids, dev_ids), store_pairs = (dev_ids, store_ids): device
        int32 tensors (engine "sm") or host lists (engine "ce"), the same pairs every layer
        (block ids are shared by all layers)."""
        self.engine = engine
        self.store, self.dev, self.L = store, dev, num_layers
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
                if self.fetch_pairs is not None:
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
                if self.store_pairs is not None:
                    self.store.store_layer(self.dev, layer, *self.store_pairs, stream=self.d2h,
                                           engine=self.engine)
                if timers is not None:
                    timers[layer][5].record(self.d2h)
        for s in (self.h2d, self.d2h, self.compute):
            cur.wait_stream(s)
