"""NEXT row F4, closed loop: Alg. 1 planned with Cost(m) from MEASURED mechanism rates
and executed by the F2 / F3 mechanisms on the GPU (Alg. 1 lines 9-18,
eqs. 28 and 35; SURVEY.md §8(f) F4 "fed by the measured H2 costs").

* ``MeasuredCosts.calibrate`` times, with CUDA events on this GPU, the two module moves
  Alg. 1 can choose -- MigrateLayer (the KV of one layer for the device's requests by
  ``bs_kv_migrate_layers`` plus the layer's weights by ``bs_copy_bytes``)
  and MigrateKVHeads (one kv-head's pages of every layer by ``bs_kv_migrate_heads_layer``,
  PAPER.md:207-212) -- and one layer's decode attention.  Cost(m) = T_transfer(m) +
  T_sync(m) (eq. 35): T_transfer = bytes / measured rate; T_sync = one measured layer of
  attention, the granularity at which the layer-wise pipeline (Fig. 6) can hand a module
  over.
* ``ModulePlacement`` records which device computes each (layer, kv-head) unit, derives
  Alg. 1's inputs (module counts, per-module load shares, costs), and executes a plan's
  moves with the mechanisms: a layer move takes d_o's highest fully-owned layer, a head
  move d_o's highest kv-head, across every layer d_o holds it for.  After the moves each
  device's pool answers for the units it owns; attention over a device's head range is
  ``bs_split_decode_attention_heads`` into disjoint rows of one output (merge = concat).

Devices here are virtual instances (pools on one GPU), as everywhere in the 1-GPU
rounds; across GPUs the pools would be peer mappings and the same calls push over NVLink.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import (KVPool, copy_bytes, kv_migrate_heads_layer, kv_migrate_layers,
               split_decode_attention_heads, split_decode_attention_heads_workspace_size)
from .policy import plan_migrations

LAYER, HEADS = 0, 1   # move kinds of bs_plan_migrations


@dataclass
class MeasuredCosts:
    """Mechanism rates measured on this GPU (bytes/s) and T_sync (s)."""
    kv_layer_Bps: float
    kv_head_Bps: float
    weight_Bps: float
    t_sync_s: float

    def layer_cost(self, kv_bytes: float, weight_bytes: float) -> float:
        """Cost(MigrateLayer) = T_transfer + T_sync (eq. 35; eq. 4's S_total / B + T_sync)."""
        return kv_bytes / self.kv_layer_Bps + weight_bytes / self.weight_Bps + self.t_sync_s

    def head_cost(self, kv_bytes: float) -> float:
        """Cost(MigrateKVHeads) = T_transfer + T_sync (eq. 35)."""
        return kv_bytes / self.kv_head_Bps + self.t_sync_s

    @classmethod
    def calibrate(cls, src: KVPool, dst: KVPool, src_ids: torch.Tensor, dst_ids: torch.Tensor,
                  weight: torch.Tensor, q: torch.Tensor, block_tables: torch.Tensor,
                  kv_split: torch.Tensor, scale: float, iters: int = 5) -> "MeasuredCosts":
        """Time each mechanism ``iters`` times (after one warm-up) on the current stream:
        one layer of KV (``bs_kv_migrate_layers``), one kv-head of one layer
        (``bs_kv_migrate_heads_layer``), ``weight`` (``bs_copy_bytes``) and one layer of
        attention over ``src`` (T_sync).  ``dst``: a scratch pool of the same geometry."""
        wdst = torch.empty_like(weight)
        B, hq, _ = q.shape
        hkv = src.num_kv_heads
        o = torch.empty(B, hq, src.head_dim, device=q.device)
        m = torch.empty(B, hq, device=q.device)
        l = torch.empty(B, hq, device=q.device)
        wsn = split_decode_attention_heads_workspace_size(src, B, hkv, hkv, hq, block_tables.shape[1])
        ws = torch.zeros(max(16, wsn), dtype=torch.uint8, device=q.device)

        def timed(fn):
            fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                fn()
            b.record()
            b.synchronize()
            return a.elapsed_time(b) * 1e-3 / iters

        n = src_ids.numel()
        t_layer = timed(lambda: kv_migrate_layers(src, dst, 0, 1, src_ids, dst_ids))
        t_head = timed(lambda: kv_migrate_heads_layer(src, dst, 0, src_ids, dst_ids, 0, 0, 1))
        t_w = timed(lambda: copy_bytes(wdst, weight))
        t_sync = timed(lambda: split_decode_attention_heads(src, 0, 0, 0, hkv, hkv, q, block_tables,
                                                            kv_split, 0, scale, o, m, l, ws))
        page = src.chunk_bytes // (2 * hkv)
        return cls(kv_layer_Bps=n * src.chunk_bytes / t_layer, kv_head_Bps=n * 2 * page / t_head,
                   weight_Bps=weight.numel() * weight.element_size() / t_w, t_sync_s=t_sync)


class ModulePlacement:
    """Which device computes each (layer, kv-head) unit, and the moves that change it.

    pools[d]: device d's KV pool (every layer / kv-head slot; only owned units are valid);
    ids[d]: int32 device tensor, the block ids of the requests' blocks in pools[d], in one
    common order (block i of the requests is ids[0][i] on device 0, ids[d][i] on d);
    weights[d][l]: device d's buffer for layer l's weights (same shape on every device)."""

    def __init__(self, pools, ids, weights, owner=None):
        self.pools, self.ids, self.weights = list(pools), list(ids), weights
        self.n_dev = len(self.pools)
        self.L, self.H = self.pools[0].num_layers, self.pools[0].num_kv_heads
        self.owner = owner if owner is not None else [[0] * self.H for _ in range(self.L)]
        self.executed = []

    # ---- Alg. 1 inputs ---------------------------------------------------------------
    def units(self, d: int) -> int:
        return sum(row.count(d) for row in self.owner)

    def full_layers(self, d: int):
        return [l for l in range(self.L) if all(x == d for x in self.owner[l])]

    def heads(self, d: int):
        return [h for h in range(self.H) if any(self.owner[l][h] == d for l in range(self.L))]

    def load(self, d: int) -> float:
        """eq. 32 with compute and memory both proportional to the owned units (each unit is
        one (layer, kv-head) of attention over the same requests): U_d in [0, 2]."""
        return 2.0 * self.units(d) / (self.L * self.H)

    def plan(self, costs: MeasuredCosts, delta: float, rho: float, supports_layer=None,
             supports_attn=None, max_moves: int = 64):
        """One Alg. 1 cycle (bs_plan_migrations) with Cost(m) from ``costs``: a layer
        module moves the chunks of one layer plus its weights, a head module one
        kv-head's pages of every layer the device holds it for."""
        n = self.n_dev
        nblk = self.ids[0].numel()
        page = self.pools[0].chunk_bytes // (2 * self.H)
        wbytes = self.weights[0][0].numel() * self.weights[0][0].element_size()
        layer_load = [2.0 / self.L] * n
        head_load, head_cost = [], []
        for d in range(n):
            nl = max(1, sum(1 for l in range(self.L) if d in self.owner[l]))
            head_load.append(2.0 * nl / (self.L * self.H))
            head_cost.append(costs.head_cost(nl * nblk * 2 * page))
        layer_cost = [costs.layer_cost(nblk * self.pools[0].chunk_bytes, wbytes)] * n
        return plan_migrations([self.load(d) for d in range(n)],
                               [len(self.full_layers(d)) for d in range(n)], layer_load, layer_cost,
                               [len(self.heads(d)) for d in range(n)], head_load, head_cost,
                               supports_layer or [1] * n, supports_attn or [1] * n, delta, rho,
                               max_moves)

    # ---- execution (Alg. 1 lines 13 / 15 / 17-18) ----------------------------------------
    def execute(self, moves, stream=None) -> None:
        for kind, d_o, d_u in moves:
            if kind == LAYER:
                l = max(self.full_layers(d_o))
                kv_migrate_layers(self.pools[d_o], self.pools[d_u], l, 1, self.ids[d_o], self.ids[d_u],
                                  stream=stream)
                copy_bytes(self.weights[d_u][l], self.weights[d_o][l], stream=stream)
                self.owner[l] = [d_u] * self.H
                self.executed.append(("layer", l, d_o, d_u))
            elif kind == HEADS:
                h = max(self.heads(d_o))
                for l in range(self.L):
                    if self.owner[l][h] == d_o:
                        kv_migrate_heads_layer(self.pools[d_o], self.pools[d_u], l, self.ids[d_o],
                                               self.ids[d_u], h, h, 1, stream=stream)
                        self.owner[l][h] = d_u
                self.executed.append(("heads", h, d_o, d_u))
            else:
                raise ValueError(f"unknown move kind {kind}")

    # ---- attention over the current placement -------------------------------------------
    def head_runs(self, layer: int):
        """(device, first kv-head, count) runs of one layer's heads, in head order."""
        runs, row = [], self.owner[layer]
        for h, d in enumerate(row):
            if runs and runs[-1][0] == d and runs[-1][1] + runs[-1][2] == h:
                runs[-1][2] += 1
            else:
                runs.append([d, h, 1])
        return [tuple(r) for r in runs]

    def attention(self, layer: int, q, block_tables, kv_split, scale, o, m, l, stream=None) -> None:
        """Partial (o~, m, l) rows of every head of ``layer``, each head range computed on
        the device that owns it (block_tables[d]: device d's tables)."""
        B, hq, _ = q.shape
        for d, h0, nh in self.head_runs(layer):
            pool = self.pools[d]
            bt = block_tables[d]
            wsn = split_decode_attention_heads_workspace_size(pool, B, nh, self.H, hq, bt.shape[1])
            ws = torch.zeros(max(16, wsn), dtype=torch.uint8, device=q.device)
            split_decode_attention_heads(pool, layer, h0, h0, nh, self.H, q, bt, kv_split, 0, scale,
                                         o, m, l, ws, stream=stream)
