"""Multi-instance decode step: attention-level migration across a ring of GPUs.

Rank r is the *home* (decode) instance of its own batch and the *cold* instance of
rank prev = r-1 (mod N) (Fig. 4: KV2 "offloaded to a cold GPU"):

  home pool  (rank r): shard 0 of r's requests   + free blocks receiving hand-offs
  cold pool  (rank r): shard 1 of prev's requests + KV being handed off to prev

Per layer l (every exchange is point-to-point: pushes into peer memory with the P2P
transport, or the library's own NCCL communicator -- bs_exchange through the C-ABI --
with the NCCL transport):
  migration  : cold pool --gather--> send to prev ; recv from next --scatter--> home pool
               (H2 two-sided transport; at N=1 the fused copy kernel P -> D)
  q exchange : send q_l of my requests to next (their cold instance); recv prev's q_l
               (issued for all layers at the start of the step)
  attention  : shard 0 of my requests over the home pool               (H4)
               shard 1 of prev's requests over the cold pool (prev's q) (H4)
  exchange   : send prev's partial (o~, m, l) to prev; recv mine from next  (H5,
               PAPER.md:237 "O^(1) (or E^(2)) is sent back")
  merge      : LSE merge of my two partials -> bf16 O, fp32 lse           (H6)
Streams: compute, copy (migration, high priority) and comm (q / partial exchange +
merge), ordered by events; the attention of layer l waits for layer l's migration
(layer-wise overlap, Fig. 6).  At N=1 the ring closes on itself: no
exchange, prev = next = self, and both shards being local, attention over both pools and
the LSE merge run as ONE fused launch (bs_split_decode_attention_local).

The protocol is written against three small interfaces -- ``ops`` (the kernels), ``ex``
(streams/events) and a wire (``exchange(sends, recvs)``: transport.NcclWire on GPUs) --
so the identical code runs on GPUs with libbanaserve.so and on CPU under gloo in the
tests (where ``ops`` and the wire are test infrastructure).
"""
from __future__ import annotations

import contextlib

import numpy as np
import torch
import torch.distributed as dist

from .transport import ErrorFlag, NcclWire, nvtx


def _out_timer(timers, layer, stream):
    """Optional 5th timer of a layer: recorded where out[l] / lse[l] become final (after the
    exchange and the merge), so attn_end -> out gives the exchange + merge latency."""
    if timers is not None and len(timers[layer]) > 4:
        timers[layer][4].record(stream)


class CudaExec:
    """Streams and events on the current CUDA device."""

    def __init__(self, device):
        self.device = device
        self.compute = torch.cuda.Stream(device=device)
        self.copy = torch.cuda.Stream(device=device, priority=-1)
        self.comm = torch.cuda.Stream(device=device)

    def use(self, s):
        return torch.cuda.stream(s)

    def event(self):
        return torch.cuda.Event()

    def record(self, ev, s):
        ev.record(s)

    def wait(self, s, ev):
        if ev is not None:   # None: nothing to wait for (e.g. inputs covered by an earlier wait)
            s.wait_event(ev)

    def begin(self):
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        for s in (self.compute, self.copy, self.comm):
            s.wait_event(ev)

    def end(self):
        cur = torch.cuda.current_stream()
        for s in (self.compute, self.copy, self.comm):
            cur.wait_stream(s)


class CpuExec:
    """Sequential execution (gloo tests): streams and events are no-ops."""
    compute = copy = comm = None

    def use(self, s):
        return contextlib.nullcontext()

    def event(self):
        return None

    def record(self, ev, s):
        pass

    def wait(self, s, ev):
        pass

    def begin(self):
        pass

    def end(self):
        pass


class CudaOps:
    """The kernels: C-ABI calls into libbanaserve.so on the current stream."""

    def __init__(self, scale: float):
        from . import (kv_gather_layer, kv_migrate_layer, kv_scatter_layer, merge_partials,
                       split_decode_attention)
        self._att, self._merge = split_decode_attention, merge_partials
        self._mig, self._gather, self._scatter = kv_migrate_layer, kv_gather_layer, kv_scatter_layer
        self.scale = scale

    def attention(self, pool, layer, q, block_tables, kv_split, shard_id, part):
        o, m, l, ws = part[:4]
        self._att(pool, layer, q, block_tables, kv_split, shard_id, self.scale, o, m, l, ws)

    def merge(self, parts, out, lse):
        self._merge([p[0] for p in parts], [p[1] for p in parts], [p[2] for p in parts], out, lse)

    def attention_local(self, pools, layer, q, block_tables, shard_ids, kv_split, out, lse, ws,
                        pdl=False):
        """H4 + H6 fused over shards resident on this GPU (one launch).  pdl: the previous
        kernel on the stream is the previous layer's attention (nothing it writes is read
        before the launch's griddepcontrol.wait) -> programmatic dependent launch."""
        from . import ATTN_PDL, split_decode_attention_local
        split_decode_attention_local(pools, layer, q, block_tables, shard_ids, kv_split,
                                     self.scale, out, lse, ws, flags=ATTN_PDL if pdl else 0)

    def local_workspace(self, pools, block_tables, batch, hq, device):
        from . import split_decode_attention_local_workspace_size
        n = split_decode_attention_local_workspace_size(pools, [t.shape[1] for t in block_tables],
                                                        batch, hq)
        return torch.zeros(max(n, 16), dtype=torch.uint8, device=device)

    def attention_tasks(self, problems, tasks, layer, batch, hq):
        """H4 + H5 + H6 fused across GPUs: partials go straight into each problem's home
        workspace (peer-mapped), the last-arriving CTA merges (one launch)."""
        from . import split_decode_attention_tasks
        split_decode_attention_tasks(problems, tasks, layer, batch, hq, self.scale)

    def problem_workspace_size(self, batch, hq, hkv, head_dim, max_blocks):
        from . import attention_problem_workspace_size
        return attention_problem_workspace_size(batch, hq, hkv, head_dim, max_blocks)

    def migrate_local(self, src, dst, layer, src_ids, dst_ids, host_ids=None):
        """Local hand-off copy: the copy kernel (SMs) or, with host id lists, the copy
        engines (DMA, no SM time -- the attention launch keeps every SM)."""
        if host_ids is not None:
            from . import kv_migrate_layer_ce
            kv_migrate_layer_ce(src, dst, layer, host_ids[0], host_ids[1])
        else:
            self._mig(src, dst, layer, src_ids, dst_ids)

    def migrate_append(self, src, dst, layer, src_ids, dst_ids, app_pool, k_new, v_new,
                       block_tables, pos):
        """H2 + H7 as one launch (N=1 migration stream)."""
        from . import kv_migrate_append_layer
        kv_migrate_append_layer(src, dst, layer, src_ids, dst_ids, app_pool, k_new, v_new,
                                block_tables, pos)

    def append(self, pool, layer, k_new, v_new, block_tables, pos):
        """H7: the decoded token's K/V into its shard's block (one launch)."""
        from . import kv_append_token
        kv_append_token(pool, layer, k_new, v_new, block_tables, pos)

    def gather(self, pool, layer, ids, staging):
        self._gather(pool, layer, ids, staging)

    def scatter(self, pool, layer, ids, staging):
        self._scatter(pool, layer, ids, staging)

    def partial_buffers(self, pool, batch, hq, head_dim, max_blocks, device):
        from . import split_decode_attention_workspace_size
        flat = torch.empty(batch * hq * (head_dim + 2), dtype=torch.float32, device=device)
        ws_n = split_decode_attention_workspace_size(pool, batch, hq, max_blocks)
        ws = torch.zeros(max(ws_n, 16), dtype=torch.uint8, device=device)
        return split_partial(flat, batch, hq, head_dim) + (ws, flat)


def split_partial(flat: torch.Tensor, batch: int, hq: int, d: int):
    """One contiguous fp32 buffer [o (B*Hq*d) | m (B*Hq) | l (B*Hq)] -> (o, m, l) views, so
    a partial crosses the wire as a single message."""
    n = batch * hq
    o = flat[: n * d].view(batch, hq, d)
    m = flat[n * d: n * d + n].view(batch, hq)
    l = flat[n * d + n: n * d + 2 * n].view(batch, hq)
    return o, m, l


def _sendrecv(wire, send: torch.Tensor, to: int, recv: torch.Tensor, frm: int):
    """One grouped send+recv (ring neighbours; symmetric on every rank => no deadlock)."""
    wire.exchange([(send, to)], [(recv, frm)])


def _all_ranks_true(flag: bool, pg, device) -> bool:
    """Logical AND over the ranks of pg (gloo: CPU tensor; NCCL: device tensor)."""
    t = torch.tensor([1 if flag else 0], dtype=torch.int32)
    if dist.get_backend(pg) != "gloo":
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=pg)
    return bool(int(t.item()))


class P2PLinks:
    """CUDA-IPC links to the two ring neighbours for the P2P transport: this rank's
    receive buffers and flags are exported; the neighbours' are mapped into this process.

    Pushes (all on this rank's streams, straight into peer memory -- no staging):
      my q[l]                      -> next.q_prev[l]       then next.flag(q, l) = epoch
      prev's shard-1 partial [l]   -> prev.part_recv[l]    then prev.flag(part, l) = epoch
      hand-off chunks (cold pool)  -> prev.home pool (the copy kernel writes the remote
                                      view directly)       then prev.flag(mig, l) = epoch
    Acks (back-pressure before a buffer is reused next step): q_ack, part_ack.

    With ``fused`` (the fused exchange): this rank's attention problem -- out, lse, the
    per-layer workspaces and `done` counters -- is exported too, and the predecessor's is
    mapped: the cold-shard CTAs write prev's partials into prev's workspace and the last
    arriver merges into prev's out / lse (no partial push, no merge launch)."""
    KINDS = ("mig", "q", "part", "q_ack", "part_ack")

    def __init__(self, rank, world, num_layers, home_pool, q_like, part_numel, handoff_dst_ids,
                 device, group, timeout_ms=20000, fused=None, kv_like=None):
        from . import ipc_export, ipc_import, pool_view
        self.L = num_layers
        self.flags = torch.zeros(len(self.KINDS) * num_layers, dtype=torch.int32, device=device)
        self.err = ErrorFlag()   # timeout flag of every wait kernel (pinned host int32)
        # device step counter: every flag value / wait target is computed from it on the
        # device, so a step captured in a CUDA graph replays with the right epoch
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.q_prev = torch.empty_like(q_like)
        self.part_recv = torch.empty((num_layers, part_numel), dtype=torch.float32, device=device)
        self.timeout_ns = int(timeout_ms) * 1_000_000
        # H7: prev's decoded-token K/V rows [L][2][B][Hkv][d], pushed with its q
        self.kv_prev = None if kv_like is None else torch.empty_like(kv_like)
        mine = {"flags": ipc_export(self.flags), "q_prev": ipc_export(self.q_prev),
                "part_recv": ipc_export(self.part_recv), "home": ipc_export(home_pool.data),
                "home_blocks": home_pool.num_blocks, "device": torch.cuda.current_device(),
                "handoff_dst": [int(x) for x in handoff_dst_ids.cpu().tolist()]}
        if self.kv_prev is not None:
            mine["kv_prev"] = ipc_export(self.kv_prev)
        if fused is not None:
            for k in ("out", "lse", "ws", "done"):
                mine[k] = ipc_export(fused[k])
            mine["ws_stride"] = fused["ws"].shape[1]
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        prev, nxt = (rank - 1) % world, (rank + 1) % world
        self._opened = {}

        def open_(who, name):
            key = (who, name)
            if key not in self._opened:
                h, off = everyone[who][name]
                self._opened[key] = (ipc_import(h, off), off)
            return self._opened[key][0]
        self.next_q_prev = open_(nxt, "q_prev")
        self.next_kv_prev = open_(nxt, "kv_prev") if self.kv_prev is not None else None
        self.next_flags = open_(nxt, "flags")
        self.prev_part_recv = open_(prev, "part_recv")
        self.prev_flags = open_(prev, "flags")
        prev_home = open_(prev, "home")
        # the view's device is the OWNER's ordinal: a push into another GPU's pool is sized
        # for NVLink (bs_kv_migrate_layer caps its CTAs), a same-GPU view is a local copy
        self.prev_home = pool_view(home_pool.num_layers, everyone[prev]["home_blocks"],
                                   home_pool.num_kv_heads, home_pool.head_dim, prev_home,
                                   everyone[prev]["device"])
        self.prev_handoff_dst = torch.tensor(everyone[prev]["handoff_dst"], dtype=torch.int32,
                                             device=device)
        self.fused = fused
        if fused is not None:  # prev's problem buffers (raw peer addresses)
            self.prev_out, self.prev_lse = open_(prev, "out"), open_(prev, "lse")
            self.prev_ws, self.prev_done = open_(prev, "ws"), open_(prev, "done")
            self.prev_ws_stride = everyone[prev]["ws_stride"]

    def flag(self, base: int, kind: str, layer: int) -> int:
        return base + 4 * (self.KINDS.index(kind) * self.L + layer)

    def my_flag(self, kind, layer):
        return self.flag(self.flags.data_ptr(), kind, layer)

    def check(self):
        self.err.check("P2P transport")

    def close(self):
        from . import ipc_close
        for ptr, off in self._opened.values():
            try:
                ipc_close(ptr, off)
            except Exception:
                pass
        self._opened = {}


class ShardedDecodeStep:
    def __init__(self, ops, ex, rank: int, world: int, home_pool, home_bt, cold_pool, cold_bt,
                 kv_split, num_q_heads: int, num_layers: int, head_dim: int,
                 handoff_src_ids=None, handoff_dst_ids=None, chunk_bytes: int = 0,
                 pg_attn=None, pg_mig=None, lookahead: int = 1, device=None,
                 fuse_local: bool = True, copy_engine: bool = False, transport: str = "nccl",
                 fused_exchange: bool = True, append=None, wire_attn=None, wire_mig=None):
        """``wire_attn`` / ``wire_mig``: the byte movers of the NCCL transport (q, K/V and
        partials on the comm stream; hand-off chunks on the copy stream) -- by default two
        transport.NcclWire communicators of the library (C-ABI), created collectively when
        the step resolves to the NCCL transport."""
        self.ops, self.ex = ops, ex
        self.rank, self.world = rank, world
        self.prev, self.next = (rank - 1) % world, (rank + 1) % world
        self.home, self.home_bt = home_pool, home_bt
        self.cold, self.cold_bt = cold_pool, cold_bt
        self.kv_split = kv_split
        # the cold pool holds shard 1 of prev's requests: index them with prev's split
        self.kv_split_cold = kv_split
        if world > 1:
            host = kv_split.cpu().numpy() if isinstance(kv_split, torch.Tensor) else kv_split
            everyone = [None] * world
            dist.all_gather_object(everyone, host.tolist(), group=pg_attn)
            if isinstance(kv_split, torch.Tensor):
                self.kv_split_cold = torch.tensor(everyone[(rank - 1) % world], dtype=kv_split.dtype,
                                                  device=kv_split.device)
            else:
                self.kv_split_cold = np.asarray(everyone[(rank - 1) % world], dtype=host.dtype)
        self.L, self.hq, self.d = num_layers, num_q_heads, head_dim
        self.B = kv_split.shape[0]
        self.src_ids, self.dst_ids = handoff_src_ids, handoff_dst_ids
        self.n_handoff = 0 if handoff_src_ids is None else int(handoff_src_ids.numel())
        # N=1 hand-off on the copy engines (host id lists) instead of the copy kernel
        self.ce_ids = None
        if copy_engine and world == 1 and self.n_handoff:
            self.ce_ids = (handoff_src_ids.cpu().tolist(), handoff_dst_ids.cpu().tolist())
        self.pg_attn, self.pg_mig = pg_attn, pg_mig
        self.lookahead = lookahead
        # H7: ``append`` = kv_new [L][2][B][Hkv][d] bf16, the decoded token's K/V of this
        # rank's requests.  The token sits at the end of shard 1 -- this rank's cold pool at
        # N=1, the next rank's cold pool at N>1 (pushed there with q) -- or, for a request
        # whose shard 1 is empty, at the end of shard 0 in this rank's home pool.
        self.append = append
        if append is not None:
            ksh = (kv_split.cpu().numpy() if isinstance(kv_split, torch.Tensor) else
                   np.asarray(kv_split)).astype(np.int64)
            l0, l1 = ksh[:, 1] - ksh[:, 0], ksh[:, 2] - ksh[:, 1]
            i32 = lambda x: torch.as_tensor(x.astype(np.int32), device=device)  # noqa: E731
            self.pos_tail = i32(np.where(l1 > 0, l1 - 1, -1))         # my requests, shard 1
            self.pos_home = i32(np.where(l1 > 0, -1, l0 - 1)) if (l1 == 0).any() else None
            if world > 1:
                kc = self.kv_split_cold
                kc = (kc.cpu().numpy() if isinstance(kc, torch.Tensor) else np.asarray(kc)).astype(np.int64)
                c1 = kc[:, 2] - kc[:, 1]
                self.pos_prev = i32(np.where(c1 > 0, c1 - 1, -1))     # prev's requests, my cold
            # NCCL transport: prev's token K/V arrive with its q (torch.distributed P2P)
            self.kv_prev_buf = torch.empty_like(append) if world > 1 else None
        dev = device
        # N=1: both shards are local -> one fused attention + merge launch per layer
        self.fuse_local = fuse_local and world == 1 and hasattr(ops, "attention_local")
        mk = lambda pool, bt: ops.partial_buffers(pool, self.B, self.hq, self.d, bt.shape[1], dev)
        # per-layer partial buffers: the merge of layer l may trail the attention of l+1
        # (not needed by the fused local launch, which merges in its epilogue)
        n_part = 0 if self.fuse_local else num_layers
        self.part_own = [mk(home_pool, home_bt) for _ in range(n_part)]
        self.part_cold = [mk(cold_pool, cold_bt) for _ in range(n_part)]
        self.part_recv = self.part_cold if world == 1 else [
            self._recv_buffer(p[4]) for p in self.part_cold]
        self.q_prev = None
        if world > 1:
            self.q_prev = None  # allocated lazily with q's shape/dtype
            nbytes = self.n_handoff * chunk_bytes
            self.stage_send = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
            self.stage_recv = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        if self.fuse_local:
            self.local_ws = ops.local_workspace([home_pool, cold_pool], [home_bt, cold_bt], self.B,
                                                self.hq, dev)
        # N>1 transport: "nccl" (torch.distributed P2P; gather/send/recv/scatter for the
        # hand-off) or "p2p" (CUDA IPC pushes straight into the neighbours' memory + flags)
        self.transport = transport if world > 1 else "local"
        self.links = None
        self.epoch = 0
        self.fused_exchange = False
        if self.transport == "p2p":
            pn = self.part_cold[0][4].numel()
            fused = None
            if fused_exchange and hasattr(ops, "attention_tasks"):
                # my problem: shard 0 on my home pool, shard 1 on next's cold pool; every
                # rank must plan it identically -> exchange the block-table widths first
                widths = [None] * world
                dist.all_gather_object(widths, (int(home_bt.shape[1]), int(cold_bt.shape[1])),
                                       group=pg_attn)
                self.mb_mine = [widths[rank][0], widths[self.next][1]]
                self.mb_prev = [widths[self.prev][0], widths[rank][1]]
                nws = ops.problem_workspace_size(self.B, num_q_heads, home_pool.num_kv_heads,
                                                 head_dim, self.mb_mine)
                # my problem is planned here (shard 0) and on next (shard 1): both must cut
                # the same ranges (the library plans from rank-invariant inputs); check it
                nws_prev = ops.problem_workspace_size(self.B, num_q_heads, home_pool.num_kv_heads,
                                                      head_dim, self.mb_prev)
                sizes = [None] * world
                dist.all_gather_object(sizes, (int(nws), int(nws_prev)), group=pg_attn)
                bad = [r for r in range(world) if sizes[(r + 1) % world][1] != sizes[r][0]]
                if bad:  # every rank sees the same list: all raise together
                    raise RuntimeError(f"problems {bad} planned differently by their home and "
                                       f"cold ranks: {sizes}")
                fused = {"out": torch.empty((num_layers, self.B, num_q_heads, head_dim),
                                            dtype=torch.bfloat16, device=dev),
                         "lse": torch.empty((num_layers, self.B, num_q_heads), dtype=torch.float32,
                                            device=dev),
                         "ws": torch.zeros((num_layers, (max(nws, 1) + 255) // 256 * 256),
                                           dtype=torch.uint8, device=dev),  # 256-B aligned rows
                         "done": torch.zeros(num_layers, dtype=torch.int32, device=dev)}
            ok, why = True, ""
            try:
                self.links = P2PLinks(rank, world, num_layers, home_pool,
                                      torch.empty((num_layers, self.B, num_q_heads, head_dim),
                                                  dtype=torch.bfloat16, device=dev),
                                      pn, handoff_dst_ids if handoff_dst_ids is not None else
                                      torch.zeros(0, dtype=torch.int32), dev, pg_attn,
                                      fused=fused, kv_like=append)
            except Exception as e:  # e.g. no peer access between these GPUs
                ok, why = False, repr(e)
            # every rank must take the same transport: fall back to NCCL unless all mapped
            if not _all_ranks_true(ok, pg_attn, dev):
                if self.links is not None:
                    self.links.close()
                self.links = None
                self.transport = "nccl"
                self.fallback_reason = why or "a peer could not map the IPC buffers"
        self.wire_attn, self.wire_mig = wire_attn, wire_mig
        if self.transport == "nccl":  # every rank takes this branch together (collective)
            if self.wire_attn is None:
                self.wire_attn = NcclWire(pg_attn)
            if self.wire_mig is None:
                self.wire_mig = NcclWire(pg_mig)
        if self.transport == "p2p":
            self.part_recv = [split_partial(self.links.part_recv[layer], self.B, self.hq, self.d)
                              + (None, self.links.part_recv[layer]) for layer in range(num_layers)]
            self.q_prev = self.links.q_prev
            self.push = torch.cuda.Stream(device=dev)
            self.merge_s = torch.cuda.Stream(device=dev)
            self.app_s = torch.cuda.Stream(device=dev)  # H7 appends (wait for prev's push)
            self.fused_exchange = self.links.fused is not None
            if self.fused_exchange:
                self.hkv = home_pool.num_kv_heads
        self.ev = {k: [ex.event() for _ in range(num_layers)]
                   for k in ("mig_done", "layer_start", "q_ready", "part_ready", "app_done")}
        self.out_ready = [ex.event() for _ in range(num_layers)]

    def _recv_buffer(self, like: torch.Tensor):
        flat = torch.empty_like(like)
        return split_partial(flat, self.B, self.hq, self.d) + (None, flat)

    @property
    def launches_per_step(self) -> int:
        """Our kernels per step, per layer: the fused local attention (N=1) or 2 attention
        launches + 1 merge; + the hand-off copy (1 kernel; gather + scatter with NCCL);
        + 8 signal / wait kernels of the P2P protocol."""
        mig = 0 if self.n_handoff == 0 or self.ce_ids is not None else (
            1 if self.world == 1 or self.transport == "p2p" else 2)
        app = 0 if self.append is None else 1 + (self.pos_home is not None)
        if (self.world == 1 and app and self.n_handoff and self.ce_ids is None
                and hasattr(self.ops, "migrate_append")):
            app -= 1   # the tail append rides the hand-off copy launch
        if self.transport == "p2p" and self.fused_exchange:
            # 1 fused attention launch; q push + signal, hand-off signal, 1 combined wait,
            # q-ack signal, done wait (per layer); H7: q-flag wait + append(s)
            # (+1 per step: the device epoch advance)
            return self.L * (1 + mig + 6 + (app + 1 if app else 0)) + 1
        if self.transport == "p2p":  # + the tiny signal / wait kernels of the protocol
            return self.L * (3 + mig + 8 + app) + 1
        attn = 1 if self.fuse_local else 3
        return self.L * (attn + mig + app)  # N>1 NCCL: the appends run on the compute stream

    def _migrate(self, layer, mig_s, timers, inputs_ready=None) -> None:
        """H2 of one layer on stream ``mig_s``: the hand-off (N=1: local copy kernel; N>1
        NCCL transport: gather -> send/recv -> scatter), then its ``mig_done`` event."""
        ex, ops, E = self.ex, self.ops, self.ev
        with ex.use(mig_s):
            if timers is not None:
                timers[layer][2].record(mig_s)
            # (layer 0 with host inputs: the hand-off copy needs none of them, so it runs
            # while they are still in flight and only the append waits -- e2e)
            fused_app = (self.world == 1 and self.append is not None and self.n_handoff > 0
                         and self.ce_ids is None and hasattr(ops, "migrate_append")
                         and not (inputs_ready is not None and layer == 0))
            if fused_app:  # H2 + H7 in one launch (the append needs this layer's inputs)
                if inputs_ready is not None:
                    ex.wait(mig_s, inputs_ready[layer])
                kv = self.append[layer]
                ops.migrate_append(self.cold, self.home, layer, self.src_ids, self.dst_ids,
                                   self.cold, kv[0], kv[1], self.cold_bt, self.pos_tail)
            elif self.n_handoff:
                if self.world == 1:
                    ops.migrate_local(self.cold, self.home, layer, self.src_ids, self.dst_ids,
                                      self.ce_ids)
                else:
                    ops.gather(self.cold, layer, self.src_ids, self.stage_send)
                    _sendrecv(self.wire_mig, self.stage_send, self.prev, self.stage_recv, self.next)
                    ops.scatter(self.home, layer, self.dst_ids, self.stage_recv)
            if self.append is not None and self.world == 1:  # H7 rides the migration stream:
                kv = self.append[layer]                      # attention waits for mig_done
                if inputs_ready is not None and not fused_app:
                    ex.wait(mig_s, inputs_ready[layer])
                if not fused_app:
                    ops.append(self.cold, layer, kv[0], kv[1], self.cold_bt, self.pos_tail)
                if self.pos_home is not None:
                    ops.append(self.home, layer, kv[0], kv[1], self.home_bt, self.pos_home)
            if timers is not None:
                timers[layer][3].record(mig_s)
            ex.record(E["mig_done"][layer], mig_s)

    def enqueue(self, q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None = None,
                timers=None, inputs_ready=None) -> None:
        """q [L][B][Hq][d] bf16 of this rank's requests -> out [L][B][Hq][d] bf16 and
        lse [L][B][Hq] fp32.  ``timers[l]`` = (attn_start, attn_end, mig_start, mig_end[,
        out_final]) events recorded on the launching streams (CUDA only).  ``inputs_ready[l]``: an
        event the step waits for before reading q[l] (e.g. its H2D copy); after the call,
        ``self.out_ready[l]`` is recorded once out[l] / lse[l] are final (per-layer D2H)."""
        with nvtx(f"banaserve step r{self.rank} n{self.world} {self.transport}"):
            return self._enqueue(q, out, lse, timers, inputs_ready)

    def _enqueue(self, q, out, lse, timers, inputs_ready):
        if self.transport == "p2p":
            self.links.check()   # a timed-out wait of an earlier step poisons its outputs
            if self.fused_exchange:
                return self._enqueue_p2p_fused(q, out, lse, timers, inputs_ready)
            return self._enqueue_p2p(q, out, lse, timers, inputs_ready)
        ex, ops, E = self.ex, self.ops, self.ev
        if self.world > 1 and (self.q_prev is None or self.q_prev.shape != q.shape):
            self.q_prev = torch.empty_like(q)
        ex.begin()
        if self.world > 1:
            # q of my requests to their cold instance (next), prev's q from prev: issued
            # up front in layer order; attention on the cold pool waits per layer
            with ex.use(ex.comm):
                for layer in range(self.L):
                    if inputs_ready is not None:
                        ex.wait(ex.comm, inputs_ready[layer])
                    _sendrecv(self.wire_attn, q[layer], self.next, self.q_prev[layer], self.prev)
                    if self.append is not None:  # H7: the token's K/V travel with q
                        _sendrecv(self.wire_attn, self.append[layer], self.next,
                                  self.kv_prev_buf[layer], self.prev)
                    ex.record(E["q_ready"][layer], ex.comm)
        # lookahead -2 at N=1: the hand-off copy runs on the compute stream right before its
        # layer's attention (serial) -- both are HBM-bound on one GPU
        mig_s = ex.compute if (self.lookahead == -2 and self.world == 1) else ex.copy
        # lookahead -3 at N=1: every layer's hand-off copy first (back to back on the copy
        # stream, per-layer events as usual), the attention of layer 0 after the last one --
        # one read/write phase, then pure-read attention
        copies_first = self.lookahead == -3 and self.world == 1 and self.n_handoff > 0
        if copies_first:
            for layer in range(self.L):
                self._migrate(layer, ex.copy, timers, inputs_ready)
        for layer in range(self.L):
            # ---- H2/H3: migration channel ---------------------------------------------
            if not copies_first:
                if self.lookahead >= 0 and layer - self.lookahead >= 0:
                    with ex.use(ex.copy):
                        ex.wait(ex.copy, E["layer_start"][layer - self.lookahead])
                self._migrate(layer, mig_s, timers, inputs_ready)
            # ---- H4: attention over both pools -------------------------------------------
            with ex.use(ex.compute):
                ex.record(E["layer_start"][layer], ex.compute)
                ex.wait(ex.compute, E["mig_done"][self.L - 1 if copies_first and layer == 0 else layer])
                if inputs_ready is not None:
                    ex.wait(ex.compute, inputs_ready[layer])
                if timers is not None:
                    timers[layer][0].record(ex.compute)
                if self.fuse_local:
                    # PDL: on the compute stream only the previous layer's attention precedes
                    # this launch (the hand-off / H7 writes are joined by the mig_done event;
                    # not with the serial schedule, lookahead -2, where the copy precedes it)
                    ops.attention_local([self.home, self.cold], layer, q[layer],
                                        [self.home_bt, self.cold_bt], [0, 1], self.kv_split,
                                        out[layer], None if lse is None else lse[layer],
                                        self.local_ws, pdl=layer > 0 and mig_s is not ex.compute)
                    if timers is not None:
                        timers[layer][1].record(ex.compute)
                    ex.record(self.out_ready[layer], ex.compute)
                    _out_timer(timers, layer, ex.compute)
                    continue
                if self.append is not None and self.world > 1 and self.pos_home is not None:
                    ops.append(self.home, layer, self.append[layer][0], self.append[layer][1],
                               self.home_bt, self.pos_home)
                ops.attention(self.home, layer, q[layer], self.home_bt, self.kv_split, 0,
                              self.part_own[layer])
                if self.world > 1:
                    ex.wait(ex.compute, E["q_ready"][layer])
                    if self.append is not None:  # H7: prev's tokens end its shard 1 here
                        kv = self.kv_prev_buf[layer]
                        ops.append(self.cold, layer, kv[0], kv[1], self.cold_bt, self.pos_prev)
                qc = q[layer] if self.world == 1 else self.q_prev[layer]
                ops.attention(self.cold, layer, qc, self.cold_bt, self.kv_split_cold, 1,
                              self.part_cold[layer])
                if timers is not None:
                    timers[layer][1].record(ex.compute)
                ex.record(E["part_ready"][layer], ex.compute)
            # ---- H5 exchange + H6 merge -------------------------------------------------
            if self.world == 1:
                with ex.use(ex.compute):
                    ops.merge([self.part_own[layer], self.part_cold[layer]], out[layer],
                              None if lse is None else lse[layer])
                    ex.record(self.out_ready[layer], ex.compute)
                    _out_timer(timers, layer, ex.compute)
            else:
                with ex.use(ex.comm):
                    ex.wait(ex.comm, E["part_ready"][layer])
                    _sendrecv(self.wire_attn, self.part_cold[layer][4], self.prev,
                              self.part_recv[layer][4], self.next)
                    ops.merge([self.part_own[layer], self.part_recv[layer]], out[layer],
                              None if lse is None else lse[layer])
                    ex.record(self.out_ready[layer], ex.comm)
                    _out_timer(timers, layer, ex.comm)
        ex.end()

    def close(self):
        """Unmap the neighbours' buffers and free the library's NCCL communicators (call on
        every rank, then barrier, before any rank frees memory its peers mapped)."""
        if self.links is not None:
            self.links.close()
        for name in ("wire_attn", "wire_mig"):
            w = getattr(self, name, None)
            if w is not None and hasattr(w, "close"):
                w.close()
            setattr(self, name, None)

    def outputs(self):
        """(out, lse) buffers the step merges into when the exchange is fused (peers write
        them); passing these to enqueue avoids a per-layer copy.  None otherwise."""
        if self.fused_exchange:
            return self.links.fused["out"], self.links.fused["lse"]
        return None

    def _enqueue_p2p_fused(self, q, out, lse, timers, inputs_ready):
        """N>1, fused exchange (SURVEY.md §8(e) "fused B200 variant"): per layer ONE launch
        runs shard 0 of my requests (home pool) and shard 1 of prev's (cold pool); each CTA
        writes its partial into the owning problem's workspace -- prev's through the IPC
        mapping -- and the last arriver of a (request, kv-head), on either GPU, merges into
        that problem's out / lse and bumps its `done` counter.  Remaining flags: hand-off
        arrival (mig), q arrival (q) and q-buffer reuse (q_ack); the done counters also
        guard workspace reuse across steps (target (epoch - 1) * B * Hkv).  Every flag
        value and wait target is computed on the device from the step counter
        ``links.epoch`` (advanced first), so the step can be captured in a CUDA graph."""
        from . import copy_ptr, epoch_advance, kv_migrate_layer, signals_epoch, wait_signals_epoch
        ex, ops, E, lk = self.ex, self.ops, self.ev, self.links
        F = lk.fused
        self.epoch += 1
        ep = lk.epoch.data_ptr()
        pc = self.B * self.hkv
        to, err = lk.timeout_ns, lk.err.ptr
        qb = q[0].numel() * q.element_size()
        own_out = out is not None and out.data_ptr() == F["out"].data_ptr()
        own_lse = lse is None or lse.data_ptr() == F["lse"].data_ptr()
        ob, lb = F["out"][0].numel() * 2, F["lse"][0].numel() * 4
        app = self.append
        kvb = 0 if app is None else app[0].numel() * app.element_size()
        epoch_advance(ep)   # on the current stream, before every stream forks from it
        ex.begin()
        for s_ in (self.push, self.merge_s, self.app_s):
            s_.wait_stream(torch.cuda.current_stream())
        with ex.use(ex.comm):  # q (+ H7: the token's K/V) of my requests -> next (their cold instance)
            for layer in range(self.L):
                if inputs_ready is not None:
                    ex.wait(ex.comm, inputs_ready[layer])
                wait_signals_epoch([lk.my_flag("q_ack", layer)], ep, 1, -1, to, err)
                copy_ptr(lk.next_q_prev + layer * qb, q[layer].data_ptr(), qb)
                if app is not None:
                    copy_ptr(lk.next_kv_prev + layer * kvb, app[layer].data_ptr(), kvb)
                signals_epoch([lk.flag(lk.next_flags, "q", layer)], ep)
        if app is not None:  # H7: prev's tokens into my cold pool, mine (empty shard 1) at home
            with torch.cuda.stream(self.app_s):
                for layer in range(self.L):
                    if self.pos_home is not None:
                        if inputs_ready is not None:
                            self.app_s.wait_event(inputs_ready[layer])
                        ops.append(self.home, layer, app[layer][0], app[layer][1], self.home_bt,
                                   self.pos_home)
                    wait_signals_epoch([lk.my_flag("q", layer)], ep, 1, 0, to, err)
                    kv = lk.kv_prev[layer]
                    ops.append(self.cold, layer, kv[0], kv[1], self.cold_bt, self.pos_prev)
                    E["app_done"][layer].record(self.app_s)
        for layer in range(self.L):
            with ex.use(ex.copy):  # hand-off: my cold pool -> prev's home pool, pushed
                if self.lookahead >= 0 and layer - self.lookahead >= 0:
                    ex.wait(ex.copy, E["layer_start"][layer - self.lookahead])
                if timers is not None:
                    timers[layer][2].record(ex.copy)
                if self.n_handoff:
                    kv_migrate_layer(self.cold, lk.prev_home, layer, self.src_ids,
                                     lk.prev_handoff_dst)
                signals_epoch([lk.flag(lk.prev_flags, "mig", layer)], ep)
                if timers is not None:
                    timers[layer][3].record(ex.copy)
            with ex.use(ex.compute):
                ex.record(E["layer_start"][layer], ex.compute)
                if inputs_ready is not None:
                    ex.wait(ex.compute, inputs_ready[layer])
                my_done = F["done"][layer:layer + 1].data_ptr()
                prev_done = lk.prev_done + 4 * layer
                wait_signals_epoch([lk.my_flag("mig", layer), lk.my_flag("q", layer), my_done,
                                    prev_done], ep, [1, 1, pc, pc], [0, 0, -pc, -pc], to, err)
                if app is not None:
                    ex.wait(ex.compute, E["app_done"][layer])
                if timers is not None:
                    timers[layer][0].record(ex.compute)
                mine = {"q": q[layer], "kv_split": self.kv_split, "max_blocks": self.mb_mine,
                        "out": F["out"][layer], "lse": F["lse"][layer], "workspace": F["ws"][layer],
                        "done": F["done"][layer:layer + 1], "cross_device": True}
                theirs = {"q": self.q_prev[layer], "kv_split": self.kv_split_cold,
                          "max_blocks": self.mb_prev, "out": lk.prev_out + layer * ob,
                          "lse": lk.prev_lse + layer * lb,
                          "workspace": lk.prev_ws + layer * lk.prev_ws_stride,
                          "workspace_bytes": lk.prev_ws_stride, "done": prev_done,
                          "cross_device": True}
                ops.attention_tasks([mine, theirs], [(self.home, self.home_bt, 0, 0),
                                                     (self.cold, self.cold_bt, 1, 1)],
                                    layer, self.B, self.hq)
                if timers is not None:
                    timers[layer][1].record(ex.compute)
                ex.record(E["part_ready"][layer], ex.compute)
            with torch.cuda.stream(self.push):  # prev's q[l] consumed -> ack
                self.push.wait_event(E["part_ready"][layer])
                signals_epoch([lk.flag(lk.prev_flags, "q_ack", layer)], ep)
            with torch.cuda.stream(self.merge_s):  # my out[l] final once every merge landed
                wait_signals_epoch([F["done"][layer:layer + 1].data_ptr()], ep, pc, 0, to, err)
                if not own_out:
                    out[layer].copy_(F["out"][layer])
                if not own_lse:
                    lse[layer].copy_(F["lse"][layer])
                self.out_ready[layer].record(self.merge_s)
                _out_timer(timers, layer, self.merge_s)
        cur = torch.cuda.current_stream()
        for s_ in (self.push, self.merge_s, self.app_s):
            cur.wait_stream(s_)
        ex.end()

    def _enqueue_p2p(self, q, out, lse, timers, inputs_ready):
        """N>1 over CUDA IPC: every exchange is a push into the neighbour's memory followed
        by a flag; consumers' streams wait on their local flags (epoch = the device step
        counter ``links.epoch``, so the step is graph-capturable)."""
        from . import copy_ptr, epoch_advance, kv_migrate_layer, signals_epoch, wait_signals_epoch
        ex, ops, E, lk = self.ex, self.ops, self.ev, self.links
        self.epoch += 1
        ep = lk.epoch.data_ptr()
        to, err = lk.timeout_ns, lk.err.ptr
        qb = q[0].numel() * q.element_size()
        app = self.append
        kvb = 0 if app is None else app[0].numel() * app.element_size()
        epoch_advance(ep)
        ex.begin()
        for s_ in (self.push, self.merge_s):
            s_.wait_stream(torch.cuda.current_stream())
        with ex.use(ex.comm):  # q (+ H7: the token's K/V) of my requests -> next
            for layer in range(self.L):
                if inputs_ready is not None:
                    ex.wait(ex.comm, inputs_ready[layer])
                wait_signals_epoch([lk.my_flag("q_ack", layer)], ep, 1, -1, to, err)
                copy_ptr(lk.next_q_prev + layer * qb, q[layer].data_ptr(), qb)
                if app is not None:
                    copy_ptr(lk.next_kv_prev + layer * kvb, app[layer].data_ptr(), kvb)
                signals_epoch([lk.flag(lk.next_flags, "q", layer)], ep)
        for layer in range(self.L):
            with ex.use(ex.copy):  # hand-off: my cold pool -> prev's home pool, pushed
                if self.lookahead >= 0 and layer - self.lookahead >= 0:
                    ex.wait(ex.copy, E["layer_start"][layer - self.lookahead])
                if timers is not None:
                    timers[layer][2].record(ex.copy)
                if self.n_handoff:
                    kv_migrate_layer(self.cold, lk.prev_home, layer, self.src_ids,
                                     lk.prev_handoff_dst)
                signals_epoch([lk.flag(lk.prev_flags, "mig", layer)], ep)
                if timers is not None:
                    timers[layer][3].record(ex.copy)
            with ex.use(ex.compute):
                ex.record(E["layer_start"][layer], ex.compute)
                wait_signals_epoch([lk.my_flag("mig", layer)], ep, 1, 0, to, err)  # hand-off in
                if inputs_ready is not None:
                    ex.wait(ex.compute, inputs_ready[layer])
                if timers is not None:
                    timers[layer][0].record(ex.compute)
                if app is not None and self.pos_home is not None:
                    ops.append(self.home, layer, app[layer][0], app[layer][1], self.home_bt,
                               self.pos_home)
                ops.attention(self.home, layer, q[layer], self.home_bt, self.kv_split, 0,
                              self.part_own[layer])
                wait_signals_epoch([lk.my_flag("q", layer)], ep, 1, 0, to, err)  # prev's q in
                if app is not None:  # H7: prev's tokens end its shard 1 in my cold pool
                    kv = lk.kv_prev[layer]
                    ops.append(self.cold, layer, kv[0], kv[1], self.cold_bt, self.pos_prev)
                ops.attention(self.cold, layer, self.q_prev[layer], self.cold_bt, self.kv_split_cold,
                              1, self.part_cold[layer])
                signals_epoch([lk.flag(lk.prev_flags, "q_ack", layer)], ep)
                if timers is not None:
                    timers[layer][1].record(ex.compute)
                ex.record(E["part_ready"][layer], ex.compute)
            with torch.cuda.stream(self.push):  # prev's shard-1 partial -> prev
                self.push.wait_event(E["part_ready"][layer])
                wait_signals_epoch([lk.my_flag("part_ack", layer)], ep, 1, -1, to, err)
                flat = self.part_cold[layer][4]
                copy_ptr(lk.prev_part_recv + layer * flat.numel() * 4, flat.data_ptr(),
                         flat.numel() * 4)
                signals_epoch([lk.flag(lk.prev_flags, "part", layer)], ep)
            with torch.cuda.stream(self.merge_s):  # my shard-1 partial from next -> merge
                wait_signals_epoch([lk.my_flag("part", layer)], ep, 1, 0, to, err)
                self.merge_s.wait_event(E["part_ready"][layer])
                ops.merge([self.part_own[layer], self.part_recv[layer]], out[layer],
                          None if lse is None else lse[layer])
                signals_epoch([lk.flag(lk.next_flags, "part_ack", layer)], ep)
                self.out_ready[layer].record(self.merge_s)
                _out_timer(timers, layer, self.merge_s)
        cur = torch.cuda.current_stream()
        for s_ in (self.push, self.merge_s):
            cur.wait_stream(s_)
        ex.end()

    def capture(self, q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None = None):
        """Capture one full step (all layers, every stream) into a CUDA graph; replaying it
        re-runs the step with whatever q / pools hold at replay time.  N=1, and N>1 with the
        P2P transport: its flags are computed on the device from the step counter, so
        every rank captures its own graph (after the same number of eager steps) and the
        ranks replay them together, one replay per step.  The NCCL transport is eager only."""
        if self.world != 1 and self.transport != "p2p":
            raise RuntimeError("graph capture needs the single-GPU step or the P2P transport")
        self.enqueue(q, out, lse)          # warm-up: lazy attributes, workspaces, maps
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.enqueue(q, out, lse)
        return g
