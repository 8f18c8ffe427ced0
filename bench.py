#!/usr/bin/env python
"""bench.py -- BanaServe (arXiv 2510.13223) hot path on B200: layer-wise KV migration
overlapped with 2-way split decode attention + exact LSE merge.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): Llama-2-7B shape (32 layers, 32 q/kv heads,
head_dim 128, bf16 KV), decode batch 64 at 2048 tokens.  Two serving instances --
decode D (home) and prefill P -- each own a paged pool.  Every request's KV is split
2-way (tokens [0,1024) in D, [1024,2048) offloaded to P: attention-level migration,
PAPER.md:207-237 Fig. 4).  During each decode step 3 more 2048-token requests are handed
off P -> D layer by layer on a side stream (Fig. 6; every layer's attention
waits for its own layer's migration event; the copy stream streams ahead unthrottled --
BS_LOOKAHEAD=-1, measured 5 % faster than lookahead 1 on one GPU).  At N=1 both instances share GPU 0 (virtual instances).  One step = all 32
layers of: migrate(l) || [split attention on D, on P -> LSE merge -> bf16 O].

value = decode tokens/s of the step (B / step time), inputs resident in HBM; pools are
70 GiB >> 126 MB L2, so no L2 flush is needed.  e2e = the same through host buffers
(q H2D from pinned memory and O/lse D2H every step).  The CPU oracle is timed beside
it on a bounded sample (cpu_baseline).  N>1 (torchrun): a ring of instances, one per GPU
-- rank r is home for its 64 requests and cold instance of rank r-1 (holds their shard 1
and their hand-off KV); q, partials and hand-off chunks cross NVLink every layer, pushed
straight into the neighbour's IPC-mapped memory (--transport p2p, default) or by NCCL P2P (weak scaling: per-GPU work is fixed).  See DESIGN.md §8.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "split decode-attn HBM GB/s & tokens/s; layer-wise KV migrate NVLink GB/s"
SHAPE = synth.LLAMA2_7B
BATCH, SEQ, N_SHARDS, N_HANDOFF = 64, 2048, 2, 3
WORKLOAD = ("C2: Llama-2-7B shape (L=32, Hq=Hkv=32, d=128, bf16 KV), decode B=64 x 2048 "
            "tokens, KV split 2-way decode/prefill pool, 3 x 2048-token requests handed off "
            "prefill->decode layer-wise per step, each request's decoded-token K/V appended")
FALLBACK_HBM_GBS = 6650.0


def omp_threads() -> int:
    """Threads the OpenMP oracle actually uses (OMP_NUM_THREADS, else the CPU affinity)."""
    if os.environ.get("OMP_NUM_THREADS"):
        return int(os.environ["OMP_NUM_THREADS"])
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


NVLINK_GBS_PER_DIR = 900.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(name: str = "ncu_attention.json"):
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("source")
    return None, None


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.

    Primary: NVML (nvidia-ml-py) polled every 5 ms from a host thread between __enter__
    (right before the first timed launch) and __exit__ (after the closing synchronize), so
    every sample lies inside the region.  Fallback (no NVML): nvidia-smi every 20 ms,
    started 1 s early, samples with < 50 % utilisation (before the region) dropped."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.rows = []

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(self.index)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        try:
            h = pynvml.nvmlDeviceGetHandleByPciBusId_v2(bus)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        return pynvml, h

    def _poll(self):
        nv, h = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        cmax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self.stop.is_set():
            try:
                clk = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((clk, cmax, 100.0,
                                  ["Active" if r & bits[n] else "Not Active" for n in self.NAMES]))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        import threading
        try:
            self.nvml = self._nvml_handle()
        except Exception:
            self.nvml = None
        if self.nvml is not None:
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(1.0)   # nvidia-smi is sampling before the timed region starts
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join()
            try:
                self.nvml[0].nvmlShutdown()
            except Exception:
                pass
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = self.rows
        source = "nvml (5 ms, timed region only)"
        if self.nvml is None:
            if self.proc is None:
                return None
            source = "nvidia-smi (20 ms, utilisation >= 50 %)"
            self.f.seek(0)
            for line in self.f.read().strip().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    clk, cmax = float(parts[0]), float(parts[1])
                except ValueError:
                    continue
                try:
                    util = float(parts[6]) if len(parts) > 6 else 100.0
                except ValueError:
                    util = 100.0
                rows.append((clk, cmax, util, parts[2:6]))
            os.unlink(self.f.name)
        busy = [r for r in rows if r[2] >= 50.0] or rows   # samples under load (else all)
        sm = [r[0] for r in busy]
        mx = [r[1] for r in busy]
        reasons = set()
        for r in busy:
            for n, v in zip(self.NAMES, r[3]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "sm_mhz_min": min(sm), "source": source}


# --------------------------------------------------------------------------------------
# the workload on the device
# --------------------------------------------------------------------------------------

def build_workload(bs, device, rank=0, world=1, layers=None, transport="p2p"):
    """Rank r's share of the ring (paper_2510_13223_b200/ring.py): home pool = shard 0 of
    its own 64 requests + free blocks for hand-offs; cold pool = shard 1 of rank r-1's
    requests + the KV handed off to r-1.  At N=1 the ring closes on itself."""
    import torch.distributed as dist
    from paper_2510_13223_b200.ring import CudaExec, CudaOps, ShardedDecodeStep

    L = SHAPE.n_layers if layers is None else layers
    prev = (rank - 1) % world
    lens = np.full(BATCH, SEQ, dtype=np.int64)
    ks = synth.block_aligned_split(lens, N_SHARDS)
    handoff_blocks = N_HANDOFF * synth.ceil_div(SEQ, SHAPE.bs)
    home_t, home_bt = synth.device_pool(SHAPE, ks[:, 1] - ks[:, 0], synth.shard_seed(rank, 0),
                                        device, spare_blocks=handoff_blocks, layers=L)
    cold_t, cold_bt = synth.device_pool(SHAPE, ks[:, 2] - ks[:, 1], synth.shard_seed(prev, 1),
                                        device, spare_blocks=handoff_blocks, layers=L)
    q = synth.device_q(SHAPE, BATCH, rank, device, L)
    case = synth.DeviceShards(SHAPE, lens, ks, [home_t, cold_t], [home_bt, cold_bt], q)
    pools = []
    for pt, bt in ((home_t, home_bt), (cold_t, cold_bt)):
        pool = bs.KVPool(L, pt.shape[1], SHAPE.hkv, SHAPE.d, base=pt.reshape(-1))
        # register the placement with the allocator: take everything, return the free ids
        pool.alloc(pool.num_blocks)
        used = set(int(x) for x in bt.ravel() if x >= 0)
        pool.free(sorted(set(range(pool.num_blocks)) - used))
        pools.append(pool)
    home, cold = pools
    # hand-off requests: their KV sits in the cold pool's spare blocks; home allocates
    src_ids = cold.alloc(handoff_blocks)
    assert src_ids == handoff_src_ids(case, handoff_blocks)
    dst_ids = home.alloc(handoff_blocks)
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32).to(device)
    step = ShardedDecodeStep(
        CudaOps(synth.default_scale(SHAPE.d)), CudaExec(device), rank, world, home, i32(home_bt),
        cold, i32(cold_bt), i32(ks), SHAPE.hq, L, SHAPE.d, handoff_src_ids=i32(src_ids),
        handoff_dst_ids=i32(dst_ids), chunk_bytes=home.chunk_bytes,
        pg_attn=dist.group.WORLD if world > 1 else None,
        pg_mig=dist.new_group(list(range(world))) if world > 1 else None,
        lookahead=int(os.environ.get("BS_LOOKAHEAD", "-1")), device=device, copy_engine=os.environ.get("BS_HANDOFF_CE", "0") == "1",
        transport=transport, append=append_inputs(rank, device, L) if (
            os.environ.get("BS_BENCH_APPEND", "1") == "1") else None)
    return case, pools, step, ks


def append_inputs(rank, device, L):
    """H7 inputs of the step (on by default; BS_BENCH_APPEND=0 drops H7): the decoded
    token's K/V of this rank's 64 requests for every layer, kv_new [L][2][B][Hkv][d] bf16,
    seeded; the step writes them at the end of each request's shard 1 (the cold pool of
    this rank at N=1, of the next rank at N>1) before that layer's attention."""
    g = torch.Generator(device=device)
    g.manual_seed(7777 + rank)
    return torch.randn((L, 2, BATCH, SHAPE.hkv, SHAPE.d), generator=g, device=device,
                       dtype=torch.bfloat16)


def handoff_src_ids(case, n):
    """The hand-off requests' blocks in the prefill pool P: its n lowest unused ids."""
    bt = case.block_tables[1]
    used = set(int(x) for x in bt.ravel() if x >= 0)
    return [i for i in range(case.pools[1].shape[1]) if i not in used][:n]


def attn_bytes_per_layer(ks, fused: bool = True, q_sets: int = 1):
    """Algorithmic bytes of one layer's attention: per (request, shard)
    len*2*Hkv*d*2 (KV) + 4*ceil(len/16) (block table); per request Hq*d*2 (q) and, with
    the fused launches (local shards at N=1, fused exchange at N>1), the merged bf16 O +
    fp32 lse (Hq*(d*2+4)) -- without them, each shard's fp32 partial Hq*(d+2)*4 instead.
    q_sets = 2 at N>1: the launch serves its own requests' shard 0 and the predecessor's
    shard 1, i.e. two sets of q."""
    tot = (q_sets - 1) * ks.shape[0] * SHAPE.hq * SHAPE.d * 2
    n_sh = ks.shape[1] - 1
    for b in range(ks.shape[0]):
        tot += SHAPE.hq * SHAPE.d * 2
        tot += SHAPE.hq * (SHAPE.d * 2 + 4) if fused else n_sh * SHAPE.hq * (SHAPE.d + 2) * 4
        for j in range(n_sh):
            n = int(ks[b, j + 1] - ks[b, j])
            tot += n * 2 * SHAPE.hkv * SHAPE.d * 2 + 4 * synth.ceil_div(n, SHAPE.bs)
    return tot


def step_stats(per_step):
    """Median, spread and a 95 % CI of the mean over this rank's timed steps (rank 0's
    steps; the headline ms_per_step is the max over ranks of the mean)."""
    n = len(per_step)
    if n == 0:
        return None
    mean = statistics.fmean(per_step)
    sd = statistics.stdev(per_step) if n > 1 else 0.0
    return {"median": round(statistics.median(per_step), 4), "min": round(per_step[0], 4),
            "max": round(per_step[-1], 4), "mean": round(mean, 4),
            "ci95": round(1.96 * sd / n ** 0.5, 4), "n": n,
            "note": "per-step boundaries are events on the main stream; steps overlap a little "
                    "(the copy stream runs ahead), the mean over K is the exact figure"}


def _allreduce_max(t):
    """Max over ranks (gloo needs CPU tensors, NCCL device tensors)."""
    if torch.distributed.get_backend() == "gloo":
        c = t.cpu()
        torch.distributed.all_reduce(c, op=torch.distributed.ReduceOp.MAX)
        return c
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t


def run_ours(args, rank, world, device):
    import paper_2510_13223_b200 as bs

    torch.cuda.set_device(device)
    case, pools, step, ks = build_workload(bs, device, rank, world, transport=args.transport)
    L = SHAPE.n_layers
    q = case.q
    own = step.outputs()   # fused exchange: the buffers peers merge into (no copy)
    if own is not None:
        out, lse = own
    else:
        out = torch.empty((L, BATCH, SHAPE.hq, SHAPE.d), dtype=torch.bfloat16, device=device)
        lse = torch.empty((L, BATCH, SHAPE.hq), dtype=torch.float32, device=device)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step.enqueue(q, out, lse)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    # ---- timed region: K steps, kernel events live on their launching streams --------
    K = args.steps
    timers = [[tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(L)]
              for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(K - 1)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record()
        for k in range(K):
            step.enqueue(q, out, lse, timers=timers[k])
            if k < K - 1:
                step_ev[k].record()
        t1.record()
        torch.cuda.synchronize()
    barrier()
    if step.links is not None:
        step.links.check()
    ms = t0.elapsed_time(t1) / K
    bounds = [t0] + step_ev + [t1]
    per_step = sorted(a.elapsed_time(b) for a, b in zip(bounds[:-1], bounds[1:]))
    attn_ms = [a.elapsed_time(b) for tk in timers for (a, b, _, _) in tk]
    mig_ms = [c.elapsed_time(d) for tk in timers for (_, _, c, d) in tk]
    # ---- exposure of the migration: the same steps without hand-offs --
    n_handoff, step.n_handoff = step.n_handoff, 0
    for _ in range(2):
        step.enqueue(q, out, lse)
    barrier()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(K):
        step.enqueue(q, out, lse)
    c1.record()
    torch.cuda.synchronize()
    step.n_handoff = n_handoff
    # ---- the hand-off alone (N=1: the same per-layer copy launches, nothing beside them)
    ms_mig_only = None
    if world == 1 and n_handoff:
        def mig_only():
            for layer in range(L):
                step.ops.migrate_local(step.cold, step.home, layer, step.src_ids, step.dst_ids,
                                       step.ce_ids)
        mig_only()
        torch.cuda.synchronize()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record()
        for _ in range(K):
            mig_only()
        m1.record()
        torch.cuda.synchronize()
        ms_mig_only = m0.elapsed_time(m1) / K
    ms_compute = torch.tensor([c0.elapsed_time(c1) / K], device=device)
    ms_t = torch.tensor([ms], device=device)
    if world > 1:
        ms_t = _allreduce_max(ms_t)
        ms_compute = _allreduce_max(ms_compute)
    ms_compute = float(ms_compute.item())
    ms_max = float(ms_t.item())

    # ---- e2e: same step through host buffers ----------------------------------------
    # every step: q copied H2D from pinned memory layer by layer on its own stream (layer
    # l's attention waits only for its own q), O / lse copied D2H layer by layer as each
    # layer finishes, then the host waits for the step's result (the next decode step needs
    # it).  The copies ride the copy engines under the previous/next layers' compute.
    # The step's inputs of layer l -- q_l and (H7) the decoded token's K/V kv_l -- sit
    # packed in one row [q_l | kv_l] of a pinned host buffer and of a device buffer, so each
    # layer is ONE copy; the step reads q and its append K/V as strided views of that buffer.
    kv0 = step.append
    qb = q[0].numel() * q.element_size()
    kvb = 0 if kv0 is None else kv0[0].numel() * kv0.element_size()
    rowb = qb + kvb
    in_host = torch.empty((L, rowb), dtype=torch.uint8).pin_memory()
    in_dev = torch.empty((L, rowb), dtype=torch.uint8, device=device)
    in_host[:, :qb].copy_(q.cpu().view(torch.uint8).reshape(L, qb))
    q_dev = in_dev[:, :qb].view(q.dtype).view(q.shape)
    if kv0 is not None:
        in_host[:, qb:].copy_(kv0.cpu().view(torch.uint8).reshape(L, kvb))
        step.append = in_dev[:, qb:].view(kv0.dtype).view(kv0.shape)
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    lse_host = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
    h2d = torch.cuda.Stream(device=device)
    d2h = torch.cuda.Stream(device=device)
    q_ev = [torch.cuda.Event() for _ in range(L)]
    cur = torch.cuda.current_stream()
    ob, lb = out[0].numel() * out.element_size(), lse[0].numel() * lse.element_size()

    def e2e_step():  # every copy through the library's own bs_copy_bytes (C-ABI)
        h2d.wait_stream(cur)
        for layer in range(L):
            bs.copy_ptr(in_dev.data_ptr() + layer * rowb, in_host.data_ptr() + layer * rowb, rowb,
                        stream=h2d)
            q_ev[layer].record(h2d)
        step.enqueue(q_dev, out, lse, inputs_ready=q_ev)
        for layer in range(L):
            d2h.wait_event(step.out_ready[layer])
            bs.copy_ptr(out_host.data_ptr() + layer * ob, out.data_ptr() + layer * ob, ob, stream=d2h)
            bs.copy_ptr(lse_host.data_ptr() + layer * lb, lse.data_ptr() + layer * lb, lb, stream=d2h)
        cur.wait_stream(d2h)
        cur.synchronize()  # the next decode step needs this step's result on the host

    for _ in range(2):
        e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / K], device=device)
    if world > 1:
        e2e_ms = _allreduce_max(e2e_ms)
    e2e_ms = float(e2e_ms.item())
    assert torch.equal(out_host.view(torch.int16), out.cpu().view(torch.int16))

    # ---- derived numbers ----------------------------------------------------------------
    a_bytes = attn_bytes_per_layer(ks, fused=step.fuse_local or step.fused_exchange,
                                   q_sets=2 if world > 1 else 1)
    mig_bytes = step.n_handoff * pools[0].chunk_bytes  # per layer, counted once
    attn_avg_ms = statistics.fmean(attn_ms)
    mig_avg_ms = statistics.fmean(mig_ms)
    attn_gbs = a_bytes / (attn_avg_ms * 1e-3) / 1e9
    mig_gbs = mig_bytes / (mig_avg_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic, traffic_src = ncu_traffic()
    tokens_s = BATCH * world / (ms_max * 1e-3)
    res = {
        "metric": METRIC,
        "value": round(tokens_s, 2),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max, 4),
        "step_ms_stats": step_stats(per_step),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 KV/q, Llama-2-7B shape, random-init; no weights)",
        "config": {
            "workload": WORKLOAD,
            "layers": L, "batch": BATCH, "seq_len": SEQ, "num_q_heads": SHAPE.hq,
            "num_kv_heads": SHAPE.hkv, "head_dim": SHAPE.d, "kv_shards": N_SHARDS,
            "handoff_requests_per_step": N_HANDOFF,
            "h7_append": step.append is not None, "parallelism": (f"ring of {world} instances (home + cold per GPU), {step.transport} transport"
                            + (", fused exchange (partials stored into the home GPU's workspace, "
                               "last-arriving CTA merges)" if step.fused_exchange else "")
                            + (f" (p2p unavailable: {step.fallback_reason})"
                               if getattr(step, "fallback_reason", None) else "")
                            + (" [ALL RANKS ON ONE GPU: functional check only]"
                               if os.environ.get("BS_RING_SAME_GPU") == "1" else "")
                            if world > 1 else "1 GPU, 2 virtual instances"),
            "l2": "no flush: resident pools 70 GiB >> 126 MB L2",
        },
        "attn_hbm_gbs": round(attn_gbs, 1),
        "attn_ms_per_layer": round(attn_avg_ms, 5),
        "migrate_gbs": round(mig_gbs, 1),
        "migrate_ms_per_layer": round(mig_avg_ms, 5),
        "migrate_bytes_per_layer": mig_bytes,
        "migrate_transport": ("fused copy kernel, local HBM (N=1: both instances on GPU 0)" if world == 1
                              else ("copy kernel pushing into the peer's IPC-mapped pool (P2P, NVLink)"
                                    if step.transport == "p2p" else
                                    "gather -> NCCL send/recv over NVLink -> scatter")),
        "roofline": {
            "bound": "hbm",
            "kernel": ("split_decode_attn_mma, fused local shards + LSE merge (1 launch per layer)"
                       if step.fuse_local else
                       "split_decode_attn_mma, own shard + predecessor's shard, partials into the "
                       "home GPU's workspace, last-arriving CTA merges (1 launch per layer)"
                       if step.fused_exchange else "split_decode_attn_mma (2 shard launches per layer)"),
            "achieved": round(attn_gbs, 1), "peak": peak, "peak_source": peak_src,
            "unit": "GB/s", "frac": round(attn_gbs / peak, 4),
            "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_layer": a_bytes,
        },
        # the hand-off copy kernel (H2): local HBM read + write at N=1 (sharing HBM with the
        # attention beside it), NVLink payload per direction at N>1 (spec peak, unmeasured here)
        "roofline_migrate": ({
            "bound": "hbm", "kernel": "copy_pages_vec16 (hand-off, copy stream)",
            "achieved": round(2 * mig_bytes / (mig_avg_ms * 1e-3) / 1e9, 1), "peak": peak,
            "peak_source": peak_src, "unit": "GB/s",
            "frac": round(2 * mig_bytes / (mig_avg_ms * 1e-3) / 1e9 / peak, 4),
            "note": "read + write bytes; in-step, concurrent with the HBM-bound attention",
            "traffic": ncu_traffic("ncu_copy.json")[0], "traffic_source": ncu_traffic("ncu_copy.json")[1]}
            if world == 1 else {
            "bound": "nvlink", "kernel": ("copy_pages_vec16 push into the peer's pool"
                                          if step.transport == "p2p" else "gather/NCCL/scatter"),
            "achieved": round(mig_gbs, 1), "peak": NVLINK_GBS_PER_DIR,
            "peak_source": "spec (NVLink 5: 900 GB/s per direction per GPU)", "unit": "GB/s",
            "frac": round(mig_gbs / NVLINK_GBS_PER_DIR, 4)}) if mig_bytes else None,
        "overlap": {"step_ms": round(ms_max, 4), "compute_only_ms": round(ms_compute, 4),
                    "exposure": round((ms_max - ms_compute) / ms_compute, 4),
                    "migrate_only_ms": None if ms_mig_only is None else round(ms_mig_only, 4),
                    "overlap_efficiency": (None if ms_mig_only is None else round(
                        (ms_compute + ms_mig_only - ms_max) / min(ms_compute, ms_mig_only), 4)),
                    "migrate_bytes_per_step": mig_bytes * L,
                    "note": ("N=1: the hand-off and the attention share one GPU's HBM, so the "
                             "hand-off's bytes cannot be hidden; over NVLink (N>1) its write side "
                             "leaves the GPU") if world == 1 else "N>1"},
        "gpu_launches": step.launches_per_step * K,
        "e2e": {"value": round(BATCH * world / (e2e_ms * 1e-3), 2), "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 4),
                "h2d_bytes_per_step": q.numel() * q.element_size() + (
                    0 if step.append is None else step.append.numel() * step.append.element_size()),
                "d2h_bytes_per_step": out.numel() * out.element_size() + lse.numel() * lse.element_size()},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(case, budget_s=args.cpu_seconds)
    return res


# --------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------------------

def oracle_sample(case, req_ids, layer, handoff_chunks: int):
    """Host copies for one oracle sample (inputs from the seeded generator, not kernels)."""
    sp, sbt, sks, sq = synth.extract_requests(case, req_ids, layer)
    P = case.pools[1]
    ids = torch.tensor(handoff_src_ids(case, handoff_chunks), dtype=torch.long, device=P.device)
    src = P[layer:layer + 1].index_select(1, ids).cpu().view(torch.int16).numpy().view(np.uint16)
    return sp, sbt, sks, sq, np.ascontiguousarray(src)


def time_oracle_sample(sample, scale):
    import oracle
    sp, sbt, sks, sq, src = sample
    n_chunks = src.shape[1]
    dst = np.empty_like(src)
    # H7 inputs: each sampled request's decoded token at the end of shard 1 (its stored
    # rows serve as the new K/V: data preparation, outside the timed region)
    pos = (sks[:, 2] - sks[:, 1] - 1).astype(np.int32)
    blk = sbt[1][np.arange(len(pos)), pos // 16]
    k_new = np.ascontiguousarray(sp[1][0, blk, 0, :, pos % 16, :])
    v_new = np.ascontiguousarray(sp[1][0, blk, 1, :, pos % 16, :])
    t = time.perf_counter()
    oracle.append_token(sp[1], 0, k_new, v_new, sbt[1], pos)
    parts = [oracle.attention_shard(p, 0, sq, bt, sks, j, scale) for j, (p, bt) in enumerate(zip(sp, sbt))]
    oracle.merge_partials([x[0] for x in parts], [x[1] for x in parts], [x[2] for x in parts])
    ta = time.perf_counter() - t
    t = time.perf_counter()
    oracle.migrate_layer(src, dst, 0, np.arange(n_chunks), np.arange(n_chunks))
    tm = time.perf_counter() - t
    return ta, tm


def cpu_baseline(case, budget_s=12.0, reqs_per_sample=32, n_samples=4):
    """Time the oracle (as it stands) on sampled (layer, 32-request) units -- extracted
    once, then re-timed round-robin until ~budget_s of oracle CPU time -- and extrapolate
    linearly to the full step: T = L * (B/r * t_attn + H * t_mig)."""
    import oracle
    oracle.lib()
    scale = synth.default_scale(SHAPE.d)
    handoff_chunks = synth.ceil_div(SEQ, SHAPE.bs)  # one hand-off request's chunks
    L = case.pools[0].shape[0]
    samples = []
    for i in range(n_samples):
        layer = (i * 7) % L
        req = [(i * reqs_per_sample + r) % BATCH for r in range(reqs_per_sample)]
        samples.append(oracle_sample(case, req, layer, handoff_chunks))
    ta_tot = tm_tot = 0.0
    units = 0
    while units < 1000 and ta_tot + tm_tot < budget_s:
        ta, tm = time_oracle_sample(samples[units % n_samples], scale)
        ta_tot += ta
        tm_tot += tm
        units += 1
    t_attn = ta_tot / units * (BATCH / reqs_per_sample)
    t_mig = tm_tot / units * N_HANDOFF
    t_step = SHAPE.n_layers * (t_attn + t_mig)
    # the same units on one thread (timings at 1 thread and all cores)
    threads = oracle.get_threads()
    oracle.set_threads(1)
    t1a = t1m = 0.0
    n1 = 2
    for i in range(n1):
        a, m = time_oracle_sample(samples[i % n_samples], scale)
        t1a += a
        t1m += m
    oracle.set_threads(threads)
    t_step1 = SHAPE.n_layers * (t1a / n1 * (BATCH / reqs_per_sample) + t1m / n1 * N_HANDOFF)
    return {"value": round(BATCH / t_step, 4), "unit": "tokens/s", "kind": "oracle",
            "cores": omp_threads(),
            "value_1_thread": round(BATCH / t_step1, 4),
            "nproc": os.cpu_count(), "cpu_model": cpu_model(),
            "sample": (f"{units} timed (layer, {reqs_per_sample}-request) units from {n_samples} "
                       f"extracted samples (H7 append + both shards + LSE merge) + 1 hand-off request's "
                       f"chunks each, fp64 C oracle; extrapolated linearly to B={BATCH}, "
                       f"{N_HANDOFF} hand-offs, {SHAPE.n_layers} layers"),
            "measured_seconds": round(ta_tot + tm_tot, 3)}


def run_reference(args, rank, world, device):
    """--impl reference: the CPU oracle as the reference arm, per step a bounded sample."""
    import oracle

    oracle.lib()
    # the same seeded workload, laid out by synth (torch RNG) only -- no product code
    gen_dev = device if torch.cuda.is_available() else torch.device("cpu")
    nl = 2 if torch.cuda.is_available() else 1
    lens = np.full(BATCH, SEQ, dtype=np.int64)
    ks = synth.block_aligned_split(lens, N_SHARDS)
    handoff_chunks = synth.ceil_div(SEQ, SHAPE.bs)
    case = synth.device_shards(SHAPE, lens, ks, seed=0, device=gen_dev,
                               spare_blocks=N_HANDOFF * handoff_chunks, layers=nl)
    scale = synth.default_scale(SHAPE.d)
    reqs = 32   # ~70 ms of oracle work per step on 16 cores: a stable sample, minutes at most
    samples = [oracle_sample(case, [(reqs * i + r) % BATCH for r in range(reqs)], i % nl,
                             handoff_chunks) for i in range(2)]
    for i in range(args.warmup):
        time_oracle_sample(samples[i % 2], scale)
    ta = tm = 0.0
    t0 = time.perf_counter()
    for i in range(args.steps):
        a, m = time_oracle_sample(samples[i % 2], scale)
        ta += a
        tm += m
    wall = time.perf_counter() - t0
    t_step = SHAPE.n_layers * (ta / args.steps * BATCH / reqs + tm / args.steps * N_HANDOFF)
    v = BATCH / t_step
    cores = omp_threads()
    sample = (f"per step: 1 layer x {reqs} requests (H7 append + both shards + merge) + 1 hand-off request's "
              f"chunks, fp64 C oracle; extrapolated to B={BATCH}, {N_HANDOFF} hand-offs, "
              f"{SHAPE.n_layers} layers")
    return {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "parallelism": "CPU oracle"},
            "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "kind": "oracle",
                             "cores": cores, "sample": sample},
            "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "measured_seconds": round(wall, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--transport", choices=["p2p", "nccl"], default=os.environ.get("BS_TRANSPORT", "p2p"),
                    help="N>1 exchange: CUDA-IPC pushes + flags (p2p) or torch.distributed NCCL P2P")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N>1 path on a 1-GPU box: every rank on cuda:0 (time-sliced,
    # numbers meaningless), gloo for the host plumbing, P2P transport
    same_gpu = os.environ.get("BS_RING_SAME_GPU", "0") == "1"
    device = torch.device("cuda", 0 if same_gpu else local)
    if args.impl == "reference":  # rank 0 alone runs it; other ranks exit without work
        if rank == 0:
            print(json.dumps(run_reference(args, rank, world, device)), flush=True)
        return
    if world > 1:
        torch.cuda.set_device(device)
        if same_gpu:
            args.transport = "p2p"
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=device)
    try:
        res = run_ours(args, rank, world, device)
        if rank == 0:
            print(json.dumps(res), flush=True)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
