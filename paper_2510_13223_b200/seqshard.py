"""Sequence-sharded decode step: every request's KV split W ways across W GPUs.

SURVEY.md §8(e) partitioning for the C3 (4-way, 32k context) and C4 (8-way, mixed
lengths) configurations: request i's tokens are cut into W contiguous block-aligned
ranges (kv_split[i] = [0, s_1, ..., s_{W-1}, len_i]); range r lives in rank r's pool;
request i's *home* is rank i mod W, which owns its q, merges and keeps its output
(split attention of PAPER.md:216-237 with the exact LSE merge of eq. 10, reading R-A4,
generalised from the paper's two instances to W).

Per layer l, on rank r:
  q exchange : home h's q_l goes to every other rank (each holds a range of h's requests)
  attention  : shard r of EVERY home's requests over rank r's pool          (H4)
  exchange   : shard r's partial of home h's requests -> home h             (H5)
  merge      : home h merges the W partials of its requests                 (H6)

Transports:
  "p2p"        (GPU, default) -- the fused exchange: ONE launch per layer runs the W
               tasks (shard r of each home's problem, bs_split_decode_attention_tasks);
               each CTA stores its partial straight into home h's workspace through a
               CUDA-IPC mapping and the last-arriving CTA (on any rank) merges into
               home h's out / lse and bumps h's `done` counter.  q is pushed into the
               peers' q buffers by the copy engines, with epoch flags and acks.
  "collective" (the two-sided fallback) -- q of every home to every peer, W attention
               calls writing (o~, m, l) partials, each partial sent to its home, then the
               home's merge call; the bytes move through a wire (``exchange(sends,
               recvs)``): on GPUs the library's own NCCL communicator (bs_exchange via
               transport.NcclWire), in the CPU tests a gloo wire with the oracle as the
               kernels.

Optional hand-off (C4: "each destination GPU receives 8192 tokens of migrated KV per
step"): n chunks of rank r's pool are pushed, layer by layer, into rank r+1's pool
(P2P: the copy kernel writing the peer's IPC-mapped pool + a `mig` flag the peer's
attention of that layer waits for; collective: gather -> send/recv -> scatter).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .ring import _all_ranks_true, split_partial
from .transport import ErrorFlag, NcclWire, nvtx


def _rows(x, h: int, W: int):
    """Rows h, h+W, ... of a table (torch tensor or numpy array), contiguous."""
    if isinstance(x, torch.Tensor):
        return x[h::W].contiguous()
    import numpy as np
    return np.ascontiguousarray(x[h::W])


class SeqShardedStep:
    KINDS = ("q", "q_ack", "mig")

    def __init__(self, ops, rank: int, world: int, pool, block_tables: torch.Tensor,
                 kv_split: torch.Tensor, num_q_heads: int, num_layers: int, head_dim: int,
                 num_kv_heads: int, device=None, group=None, transport: str = "p2p",
                 handoff_src_ids=None, handoff_dst_ids=None, timeout_ms: int = 20000,
                 wire=None):
        """pool: this rank's KV pool (range `rank` of every request); block_tables
        [B_total, mb] its block ids per request; kv_split [B_total, W+1] (same on every
        rank).  B_total must be a multiple of W: home h serves requests h, h+W, ...
        ``wire``: byte mover of the collective transport (default: a transport.NcclWire
        over ``group``, created collectively if the step resolves to it)."""
        self.ops, self.rank, self.world = ops, rank, world
        self.timeout_ns = int(timeout_ms) * 1_000_000
        self.pool, self.L, self.hq, self.d, self.hkv = pool, num_layers, num_q_heads, head_dim, num_kv_heads
        self.group, self.device = group, device
        Bt = int(kv_split.shape[0])
        if Bt % world:
            raise ValueError(f"{Bt} requests do not split evenly over {world} homes")
        if int(kv_split.shape[1]) != world + 1:
            raise ValueError("kv_split must have W+1 columns (one range per rank)")
        self.Bh = Bt // world
        W = world
        # rows of home h's requests (i = h, h+W, ...), as contiguous per-problem tables
        self.bt_h = [_rows(block_tables, h, W) for h in range(W)]
        self.ks_h = [_rows(kv_split, h, W) for h in range(W)]
        # dispatch order of each home's requests in this rank's task launch: longest range
        # first (LPT), so mixed lengths (C4) do not leave a long CTA for the last wave; the
        # merge order is the range order, so results do not depend on it
        import numpy as np
        ks_host = kv_split.cpu().numpy() if isinstance(kv_split, torch.Tensor) else np.asarray(kv_split)
        mine = (ks_host[:, rank + 1] - ks_host[:, rank]).astype(np.int64)
        self.order_h = []
        for h in range(W):
            o = np.argsort(-mine[h::W], kind="stable").astype(np.int32)
            self.order_h.append(torch.from_numpy(o).to(block_tables.device)
                                if isinstance(block_tables, torch.Tensor) else o)
        self.src_ids, self.dst_ids = handoff_src_ids, handoff_dst_ids
        self.n_handoff = 0 if handoff_src_ids is None else int(handoff_src_ids.numel())
        self.prev, self.next = (rank - 1) % W, (rank + 1) % W
        self.epoch = 0
        # W = 1 keeps the P2P transport's fused launch (one task, no peers): the 1-GPU
        # split-K baseline of the same shapes runs the same kernel as W > 1
        self.transport = transport
        self.fallback_reason = None
        widths = [None] * W
        if W > 1:
            dist.all_gather_object(widths, int(block_tables.shape[1]), group=group)
        else:
            widths = [int(block_tables.shape[1])]
        self.max_blocks = widths  # problem h's shard s has block-table width widths[s]
        if self.transport == "p2p":
            ok, why = True, ""
            try:
                self._setup_p2p()
            except Exception as e:  # e.g. no peer access
                ok, why = False, repr(e)
            if not (_all_ranks_true(ok, group, device) if W > 1 else ok):
                if W == 1:
                    raise RuntimeError(f"sequence-sharded step setup failed: {why}")
                self.transport, self.fallback_reason = "collective", why or "a peer could not map"
        self.wire = wire
        if self.transport == "collective":
            if self.wire is None and W > 1:
                self.wire = NcclWire(group)
            self._setup_collective()

    # ------------------------------------------------------------------ P2P (fused)
    def _setup_p2p(self):
        from . import ipc_export, ipc_import, pool_view
        W, L, Bh, hq, d, dev = self.world, self.L, self.Bh, self.hq, self.d, self.device
        nws = self.ops.problem_workspace_size(Bh, hq, self.hkv, d, self.max_blocks)
        stride = (max(nws, 1) + 255) // 256 * 256
        self.flags = torch.zeros(len(self.KINDS) * W * L, dtype=torch.int32, device=dev)
        self.err = ErrorFlag()
        self.epoch_dev = torch.zeros(1, dtype=torch.int32, device=dev)  # device step counter
        self.q_in = torch.empty((W, L, Bh, hq, d), dtype=torch.bfloat16, device=dev)
        self.out_buf = torch.empty((L, Bh, hq, d), dtype=torch.bfloat16, device=dev)
        self.lse_buf = torch.empty((L, Bh, hq), dtype=torch.float32, device=dev)
        self.ws = torch.zeros((L, stride), dtype=torch.uint8, device=dev)
        self.done = torch.zeros(L, dtype=torch.int32, device=dev)
        mine = {} if W == 1 else {
            k: ipc_export(t) for k, t in (("flags", self.flags), ("q_in", self.q_in),
                                         ("out", self.out_buf), ("lse", self.lse_buf),
                                         ("ws", self.ws), ("done", self.done),
                                         ("pool", self.pool.data))}
        mine["ws_stride"] = stride
        mine["ws_bytes"] = nws   # the range plan's size: must agree on every rank
        mine["pool_blocks"] = self.pool.num_blocks
        mine["device"] = dev.index if dev.index is not None else torch.cuda.current_device()
        mine["handoff_dst"] = ([] if self.dst_ids is None else
                               [int(x) for x in self.dst_ids.cpu().tolist()])
        everyone = [None] * W
        if W > 1:
            dist.all_gather_object(everyone, mine, group=self.group)
        else:
            everyone = [mine]
        # every rank plans every home's problem from the same rank-invariant inputs (the
        # library's fixed slot model): a mismatch would corrupt the last-arriver merge
        if len({e["ws_bytes"] for e in everyone}) != 1:
            raise RuntimeError(f"ranks planned the attention problems differently: "
                               f"{[e['ws_bytes'] for e in everyone]}")
        self._opened = []

        def open_(who, name):
            h, off = everyone[who][name]
            ptr = ipc_import(h, off)
            self._opened.append((ptr, off))
            return ptr
        self.peer = {}
        for p in range(W):
            if p == self.rank:
                self.peer[p] = {"flags": self.flags.data_ptr(), "q_in": self.q_in.data_ptr(),
                                "out": self.out_buf.data_ptr(), "lse": self.lse_buf.data_ptr(),
                                "ws": self.ws.data_ptr(), "done": self.done.data_ptr(),
                                "ws_stride": stride}
                continue
            self.peer[p] = {k: open_(p, k) for k in ("flags", "q_in", "out", "lse", "ws", "done")}
            self.peer[p]["ws_stride"] = everyone[p]["ws_stride"]
        self.next_pool = None
        if self.n_handoff:
            nxt = self.next
            base = self.pool.data.data_ptr() if nxt == self.rank else open_(nxt, "pool")
            self.next_pool = pool_view(self.L, everyone[nxt]["pool_blocks"], self.pool.num_kv_heads,
                                       self.pool.head_dim, base, everyone[nxt]["device"])
            self.next_dst = torch.tensor(everyone[nxt]["handoff_dst"], dtype=torch.int32, device=dev)
        self.ack_s = torch.cuda.Stream(device=dev)
        self.out_s = torch.cuda.Stream(device=dev)
        self.comm = torch.cuda.Stream(device=dev)
        self.copy = torch.cuda.Stream(device=dev, priority=-1)
        self.out_ready = [torch.cuda.Event() for _ in range(L)]
        self.part_ready = [torch.cuda.Event() for _ in range(L)]
        self.mig_ready = [torch.cuda.Event() for _ in range(L)]   # W = 1 hand-off

    def flag(self, who: int, kind: str, src: int, layer: int) -> int:
        """Address of flag (kind, src, layer) in rank `who`'s flag array."""
        i = (self.KINDS.index(kind) * self.world + src) * self.L + layer
        return self.peer[who]["flags"] + 4 * i

    def check(self):
        if self.transport == "p2p":
            self.err.check("sequence-sharded step")

    def close(self):
        """Unmap the peers' buffers and free the NCCL communicator (call on every rank,
        then barrier, before any rank frees the memory its peers mapped)."""
        from . import ipc_close
        for ptr, off in getattr(self, "_opened", []):
            try:
                ipc_close(ptr, off)
            except Exception:
                pass
        self._opened = []
        if getattr(self, "wire", None) is not None and hasattr(self.wire, "close"):
            self.wire.close()
            self.wire = None

    def outputs(self):
        return (self.out_buf, self.lse_buf) if self.transport == "p2p" else None

    @property
    def launches_per_step(self) -> int:
        if self.transport != "p2p":
            return self.L * (self.world + 1 + (2 if self.n_handoff else 0))
        if self.world == 1:   # attention (+ hand-off copy); + the epoch advance
            return self.L * (1 + (1 if self.n_handoff else 0)) + 1
        # attention, combined wait, q-push wait + signals, ack signals, done wait (+ hand-off
        # copy and its signal); + the device epoch advance once per step
        return self.L * (1 + 1 + 2 + 1 + 1 + (2 if self.n_handoff else 0)) + 1

    def _enqueue_p2p(self, q, out, lse, timers=None, inputs_ready=None):
        """``timers[l]`` = (attn_start, attn_end, mig_start, mig_end) events recorded on the
        launching streams; ``inputs_ready[l]``: event the step waits for before reading
        q[l] (its H2D copy); ``out_ready[l]`` is recorded once out[l] / lse[l] are final."""
        from . import copy_ptr, epoch_advance, kv_migrate_layer, signals_epoch, wait_signals_epoch
        W, r, L = self.world, self.rank, self.L
        self.epoch += 1
        ep = self.epoch_dev.data_ptr()
        to, err = self.timeout_ns, self.err.ptr
        pc = self.Bh * self.hkv
        qb = q[0].numel() * q.element_size()
        ob, lb = self.out_buf[0].numel() * 2, self.lse_buf[0].numel() * 4
        peers = [p for p in range(W) if p != r]
        cur = torch.cuda.current_stream()
        epoch_advance(ep)   # flag values / wait targets are computed from it on the device
        for s in (self.comm, self.copy, self.ack_s, self.out_s):
            s.wait_stream(cur)
        with torch.cuda.stream(self.comm):  # my q_l -> every peer's q_in[r][l]
            for layer in range(L):
                if inputs_ready is not None:
                    self.comm.wait_event(inputs_ready[layer])
                if peers:
                    wait_signals_epoch([self.flag(r, "q_ack", p, layer) for p in peers], ep, 1, -1,
                                       to, err)
                for p in peers:
                    copy_ptr(self.peer[p]["q_in"] + (r * L + layer) * qb, q[layer].data_ptr(), qb)
                if peers:
                    signals_epoch([self.flag(p, "q", r, layer) for p in peers], ep)
        compute = cur
        # W = 1: every range of every problem runs in this GPU's launch, so stream order
        # already orders the workspace reuse and the merges -- events replace the flags
        solo = W == 1
        for layer in range(L):
            if self.n_handoff:
                with torch.cuda.stream(self.copy):
                    if timers is not None:
                        timers[layer][2].record(self.copy)
                    kv_migrate_layer(self.pool, self.next_pool, layer, self.src_ids, self.next_dst)
                    if timers is not None:
                        timers[layer][3].record(self.copy)
                    if solo:
                        self.mig_ready[layer].record(self.copy)
                    else:
                        signals_epoch([self.flag(self.next, "mig", r, layer)], ep)
            if solo:
                if self.n_handoff:
                    compute.wait_event(self.mig_ready[layer])
            else:
                self._wait_inputs(layer, peers, ep, pc, to, err, compute)
            if inputs_ready is not None:
                compute.wait_event(inputs_ready[layer])
            if timers is not None:
                timers[layer][0].record(compute)
            problems = []
            for h in range(W):
                P = self.peer[h]
                problems.append({
                    "q": q[layer] if h == r else self.q_in[h, layer],
                    "kv_split": self.ks_h[h], "max_blocks": self.max_blocks,
                    "out": P["out"] + layer * ob, "lse": P["lse"] + layer * lb,
                    "workspace": P["ws"] + layer * P["ws_stride"], "workspace_bytes": P["ws_stride"],
                    "done": P["done"] + 4 * layer, "cross_device": not solo})
            with torch.cuda.stream(compute):
                if solo and hasattr(self.ops, "attention_local"):
                    # W = 1: one local problem -- the fused local path, whose launches of
                    # layers > 0 are programmatic dependents of the previous layer's and
                    # may merge through a thread-block cluster
                    if getattr(self, "_solo_ws", None) is None:
                        self._solo_ws = self.ops.local_workspace([self.pool], [self.bt_h[0]], self.Bh,
                                                                 self.hq, self.out_buf.device)
                    self.ops.attention_local([self.pool], layer, problems[0]["q"], [self.bt_h[0]], [0],
                                             self.ks_h[0], self.out_buf[layer], self.lse_buf[layer],
                                             self._solo_ws, pdl=layer > 0)
                else:
                    self.ops.attention_tasks(problems, [(self.pool, self.bt_h[h], r, h, self.order_h[h])
                                                        for h in range(W)],
                                             layer, self.Bh, self.hq)
            if timers is not None:
                timers[layer][1].record(compute)
            self.part_ready[layer].record(compute)
            if peers:
                with torch.cuda.stream(self.ack_s):  # every home's q_l consumed -> acks
                    self.ack_s.wait_event(self.part_ready[layer])
                    signals_epoch([self.flag(p, "q_ack", r, layer) for p in peers], ep)
            with torch.cuda.stream(self.out_s):  # my out_l final once all merges landed
                if solo:
                    self.out_s.wait_event(self.part_ready[layer])
                else:
                    wait_signals_epoch([self.done[layer:layer + 1].data_ptr()], ep, pc, 0, to, err)
                if out.data_ptr() != self.out_buf.data_ptr():
                    out[layer].copy_(self.out_buf[layer])
                if lse is not None and lse.data_ptr() != self.lse_buf.data_ptr():
                    lse[layer].copy_(self.lse_buf[layer])
                self.out_ready[layer].record(self.out_s)
                if timers is not None and len(timers[layer]) > 4:
                    timers[layer][4].record(self.out_s)
        for s in (self.comm, self.copy, self.ack_s, self.out_s):
            cur.wait_stream(s)

    def _wait_inputs(self, layer, peers, ep, pc, to, err, compute):
        """One wait launch before layer l's attention: every peer's q_l arrived, every
        home's workspace free (its `done` counter reached the previous step's count) and the
        predecessor's hand-off of layer l landed."""
        from . import wait_signals_epoch
        W, r = self.world, self.rank
        waits = [self.flag(r, "q", p, layer) for p in peers]
        mul, add = [1] * len(peers), [0] * len(peers)
        waits += [self.peer[h]["done"] + 4 * layer for h in range(W)]
        mul += [pc] * W
        add += [-pc] * W
        if self.n_handoff:
            waits.append(self.flag(r, "mig", self.prev, layer))
            mul.append(1)
            add.append(0)
        wait_signals_epoch(waits, ep, mul, add, to, err, stream=compute)

    # ------------------------------------------------------------------ collective
    def _setup_collective(self):
        W, L, Bh, hq, d = self.world, self.L, self.Bh, self.hq, self.d
        mk = lambda: self.ops.partial_buffers(self.pool, Bh, hq, d, int(self.bt_h[0].shape[1]),
                                              self.device)
        self.parts = [mk() for _ in range(W)]      # my shard's partial of home h's requests
        self.recv = [mk() for _ in range(W)]       # home: partial of my requests from rank s
        self.q_all = None                          # [W][B_h][Hq][d]: every home's q_l
        if self.n_handoff:
            cb = getattr(self.pool, "chunk_bytes", None) or self.pool.data[0, 0].nbytes
            nbytes = self.n_handoff * cb
            kw = {} if self.device is None else {"device": self.device}
            self.stage_send = torch.empty(max(nbytes, 16), dtype=torch.uint8, **kw)
            self.stage_recv = torch.empty(max(nbytes, 16), dtype=torch.uint8, **kw)

    def _enqueue_collective(self, q, out, lse):
        W, r = self.world, self.rank
        for layer in range(self.L):
            if self.n_handoff:  # gather -> send to next / recv from prev -> scatter
                self.ops.gather(self.pool, layer, self.src_ids, self.stage_send)
                if W > 1:
                    self.wire.exchange([(self.stage_send, self.next)], [(self.stage_recv, self.prev)])
                    self.ops.scatter(self.pool, layer, self.dst_ids, self.stage_recv)
                else:
                    self.ops.scatter(self.pool, layer, self.dst_ids, self.stage_send)
            if W > 1:  # home r's q_l to every peer, every home's q_l from it (an all-gather)
                if self.q_all is None or self.q_all.shape[1:] != q[layer].shape:
                    self.q_all = torch.empty((W,) + tuple(q[layer].shape), dtype=q.dtype,
                                             device=q.device)
                self.q_all[r].copy_(q[layer])
                peers = [p for p in range(W) if p != r]
                self.wire.exchange([(self.q_all[r], p) for p in peers],
                                   [(self.q_all[p], p) for p in peers])
                q_all = [self.q_all[h] for h in range(W)]
            else:
                q_all = [q[layer]]
            for h in range(W):
                self.ops.attention(self.pool, layer, q_all[h], self.bt_h[h], self.ks_h[h], r,
                                   self.parts[h])
            sends = [(self.parts[h][4], h) for h in range(W) if h != r]
            recvs = [(self.recv[s][4], s) for s in range(W) if s != r]
            if W > 1:
                self.wire.exchange(sends, recvs)
            got = [self.parts[r] if s == r else self.recv[s] for s in range(W)]
            self.ops.merge(got, out[layer], None if lse is None else lse[layer])

    def enqueue(self, q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None = None,
                timers=None, inputs_ready=None):
        """q [L][B_h][Hq][d] of this rank's home requests (global ids rank, rank+W, ...)
        -> out [L][B_h][Hq][d] bf16, lse [L][B_h][Hq] fp32.  ``timers`` / ``inputs_ready``:
        P2P transport only (see _enqueue_p2p)."""
        with nvtx(f"banaserve seqshard step r{self.rank} n{self.world} {self.transport}"):
            if self.transport == "p2p":
                self.check()   # a timed-out wait of an earlier step poisons its outputs
                return self._enqueue_p2p(q, out, lse, timers, inputs_ready)
            return self._enqueue_collective(q, out, lse)

    def capture(self, q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None = None):
        """One step of the P2P transport captured in a CUDA graph (flags computed on the
        device from the step counter); every rank captures after the same eager steps and
        the ranks replay together."""
        if self.transport != "p2p":
            raise RuntimeError("graph capture needs the P2P transport")
        self.enqueue(q, out, lse)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.enqueue(q, out, lse)
        return g


__all__ = ["SeqShardedStep", "split_partial"]
