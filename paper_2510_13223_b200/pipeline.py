"""H3: layer-wise overlap of KV migration with split decode attention (PAPER.md:256,
:282-293, Fig. 6 "while the GPU executes forward computation for L_i, the HtoD channel
fetches KV Cache for L_{i+1}"; here the channel is the GPU-to-GPU migration of H2).

One decode step over all layers:
  copy stream    : for each layer l: [wait compute reached layer l - lookahead]
                   migrate(l) for every migration job; record mig_done[l]
  compute stream : for each layer l: wait mig_done[l];
                   split attention over every local shard (H4) -> partials;
                   exchange (H5, identity on one GPU); LSE merge (H6) -> bf16 O.
Streams and events are torch's (plumbing); every step of the path is a C-ABI call into
libbanaserve.so.  The whole step can be captured into one CUDA graph.
"""
from __future__ import annotations

import dataclasses

import torch

from . import (kv_migrate_layer, merge_partials, split_decode_attention,
               split_decode_attention_workspace_size, KVPool, MIGRATE_AUTO)


@dataclasses.dataclass
class Shard:
    """One KV shard of a batch: the pool holding it and its device-side tables."""
    pool: KVPool
    block_tables: torch.Tensor   # int32 [B][max_blocks] (device)
    shard_id: int


@dataclasses.dataclass
class MigrationJob:
    """Chunks moving src -> dst every layer (ids are device int32 [n])."""
    src: KVPool
    dst: KVPool
    src_ids: torch.Tensor
    dst_ids: torch.Tensor
    method: int = MIGRATE_AUTO


class LayerwiseDecodeStep:
    def __init__(self, shards, kv_split: torch.Tensor, num_q_heads: int, num_layers: int,
                 scale: float, migrations=(), lookahead: int = 1, compute_stream=None,
                 copy_stream=None):
        self.shards = list(shards)
        self.kv_split = kv_split
        self.migrations = list(migrations)
        self.L = num_layers
        self.scale = float(scale)
        self.lookahead = lookahead
        dev = self.shards[0].pool.device
        B = kv_split.shape[0]
        d = self.shards[0].pool.head_dim
        self.B, self.hq, self.d = B, num_q_heads, d
        self.compute = compute_stream or torch.cuda.Stream(device=dev)
        self.copy = copy_stream or torch.cuda.Stream(device=dev, priority=-1)
        self.parts = []
        for sh in self.shards:
            o = torch.empty((B, num_q_heads, d), dtype=torch.float32, device=dev)
            m = torch.empty((B, num_q_heads), dtype=torch.float32, device=dev)
            l = torch.empty((B, num_q_heads), dtype=torch.float32, device=dev)
            ws_n = split_decode_attention_workspace_size(sh.pool, B, num_q_heads,
                                                         sh.block_tables.shape[1])
            ws = torch.zeros(max(ws_n, 16), dtype=torch.uint8, device=dev)
            self.parts.append((o, m, l, ws))
        self.mig_done = [torch.cuda.Event() for _ in range(num_layers)]
        self.layer_start = [torch.cuda.Event() for _ in range(num_layers)]
        self.step_start = torch.cuda.Event()

    @property
    def launches_per_step(self) -> int:
        per_layer = len(self.shards) + 1 + sum(1 for j in self.migrations if j.src_ids.numel() > 0)
        return per_layer * self.L

    def enqueue(self, q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None = None,
                timers=None) -> None:
        """q bf16 [L][B][Hq][d]; out bf16 [L][B][Hq][d]; lse fp32 [L][B][Hq] or None.
        Enqueues one step on (compute, copy) streams; the caller's current stream is
        joined at both ends so the step composes with surrounding work.  ``timers``:
        optional per-layer (attn_start, attn_end, mig_start, mig_end) timing events,
        recorded on the stream each kernel is launched on."""
        cur = torch.cuda.current_stream()
        self.step_start.record(cur)
        self.compute.wait_event(self.step_start)
        self.copy.wait_event(self.step_start)
        for layer in range(self.L):
            with torch.cuda.stream(self.copy):
                if self.lookahead >= 0 and layer - self.lookahead >= 0:
                    self.copy.wait_event(self.layer_start[layer - self.lookahead])
                if timers is not None:
                    timers[layer][2].record(self.copy)
                for job in self.migrations:
                    if job.src_ids.numel():
                        kv_migrate_layer(job.src, job.dst, layer, job.src_ids, job.dst_ids,
                                         method=job.method, stream=self.copy)
                if timers is not None:
                    timers[layer][3].record(self.copy)
                self.mig_done[layer].record(self.copy)
            with torch.cuda.stream(self.compute):
                self.layer_start[layer].record(self.compute)
                self.compute.wait_event(self.mig_done[layer])
                if timers is not None:
                    timers[layer][0].record(self.compute)
                for sh, (o, m, l, ws) in zip(self.shards, self.parts):
                    split_decode_attention(sh.pool, layer, q[layer], sh.block_tables,
                                           self.kv_split, sh.shard_id, self.scale, o, m, l, ws,
                                           stream=self.compute)
                if timers is not None:
                    timers[layer][1].record(self.compute)
                merge_partials([p[0] for p in self.parts], [p[1] for p in self.parts],
                               [p[2] for p in self.parts], out[layer],
                               None if lse is None else lse[layer], stream=self.compute)
        cur.wait_stream(self.compute)
        cur.wait_stream(self.copy)
