#!/usr/bin/env python
"""bench.py -- BanaServe (arXiv 2510.13223) hot path on B200: layer-wise KV migration
overlapped with split decode attention + exact LSE merge.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config auto|c2|c3|c4]
                    [--impl ours|reference] [--transport p2p|nccl]

`--gpus N` > 1 without torchrun re-launches itself under `torch.distributed.run` (N ranks,
rank r on cuda:r); under torchrun WORLD_SIZE must equal N.  Fewer visible GPUs than N is
an error (BS_RING_SAME_GPU=1: every rank on cuda:0, a labelled functional check).

Headline workload (BASELINE.json configs[1], "C2"): Llama-2-7B shape (32 layers, 32 q/kv
heads, head_dim 128, bf16 KV), decode batch 64 at 2048 tokens per GPU.  Two serving
instances -- decode D (home) and prefill P -- each own a paged pool; every request's KV is
split 2-way (tokens [0,1024) in D, [1024,2048) offloaded to P: attention-level migration,
PAPER.md:207-237 Fig. 4).  During each decode step 3 more 2048-token requests are handed
off P -> D layer by layer on a side stream (Fig. 6; every layer's attention
waits for its own layer's migration event).  At N=1 both instances share GPU 0; at N>1 a
ring of instances, one per GPU -- rank r is home for its 64 requests and cold instance of
rank r-1; q, partials and hand-off chunks cross NVLink every layer, pushed into the
neighbour's IPC-mapped memory (p2p) or through the library's NCCL communicator (nccl).
Weak scaling: per-GPU work is fixed.

`--config auto` (default) prints the C2 line and adds, under "extra_configs", the
sequence-sharded configs of SURVEY.md §8(e) at the same N: C3 (Llama-3-8B GQA, 8 x 32k
requests split N ways, merge on each request's home GPU; N=1 is the 1-GPU split-K
baseline) and, at N >= 4, C4 (Llama-2-70B shape, 256 mixed-length requests split N ways,
8192 tokens of KV handed to the next GPU per layer).  `--config c3|c4` makes one of them
the headline line instead.

value = decode tokens/s of the step (requests / step time), inputs resident in HBM; every
step reads >= 4 GiB of distinct KV >> 126 MB L2, so no L2 flush is needed.  e2e = the same
through host buffers (q H2D from pinned memory, O/lse D2H every step).  The CPU oracle is
timed beside it on a bounded sample (cpu_baseline, rank 0).  See DESIGN.md §7-8.
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
SHAPE = synth.LLAMA2_7B  # C2
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
        self.power = []          # board power (W), NVML only
        self.power_limit_w = None

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
        try:
            self.power_limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
        except Exception:
            self.power_limit_w = None
        while not self.stop.is_set():
            try:
                clk = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((clk, cmax, 100.0,
                                  ["Active" if r & bits[n] else "Not Active" for n in self.NAMES]))
                self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
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
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
               "samples": len(sm), "sm_mhz_min": min(sm), "source": source}
        if self.power:   # context for sw_power_cap: the HBM-bound step's SM clock follows it
            out["power_w_median"] = round(statistics.median(self.power), 1)
            out["power_w_max"] = round(max(self.power), 1)
            out["power_limit_w"] = self.power_limit_w
        return out


class NvlinkCounters:
    """NVLink data bytes TX / RX of this GPU (NVML field values 138 / 139, KiB, all links)
    read right before and after the timed region: an independent count of what crossed
    NVLink, to corroborate the kernel-event GB/s.  None where NVML lacks the fields."""
    FIELDS = (138, 139)  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX

    def __init__(self, index: int):
        self.h = self.nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self.h = nv.nvmlDeviceGetHandleByPciBusId_v2(bus)
            self.nv = nv
        except Exception:
            self.h = None

    def read(self):
        if self.h is None:
            return None
        try:
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, list(self.FIELDS))
            if any(v.nvmlReturn != 0 for v in vals):
                return None
            return [int(v.value.ullVal) * 1024 for v in vals]
        except Exception:
            return None

    @staticmethod
    def delta(a, b, steps):
        if a is None or b is None:
            return None
        return {"tx_bytes_per_step": (b[0] - a[0]) / steps, "rx_bytes_per_step": (b[1] - a[1]) / steps,
                "source": "NVML field values 138/139 (NVLink data TX/RX, all links), read around "
                          "the timed region"}


def _barrier(world):
    if world > 1:
        torch.distributed.barrier()


def _release(world):
    """Free the previous workload's device memory (after every rank unmapped it)."""
    import gc
    _barrier(world)
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    _barrier(world)


def _allreduce_max(t):
    """Max over ranks (gloo needs CPU tensors, NCCL device tensors)."""
    if torch.distributed.get_backend() == "gloo":
        c = t.cpu()
        torch.distributed.all_reduce(c, op=torch.distributed.ReduceOp.MAX)
        return c
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t


def _max_over_ranks(x: float, world: int, device) -> float:
    t = torch.tensor([float(x)], device=device)
    if world > 1:
        t = _allreduce_max(t)
    return float(t.item())


def _all_true(flag: bool, world: int, device) -> bool:
    if world == 1:
        return flag
    return _max_over_ranks(0.0 if flag else 1.0, world, device) == 0.0


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


class DrvTimer:
    """A timing CUDA event recorded with CU_EVENT_RECORD_EXTERNAL: inside a stream capture
    it becomes an event-record NODE of the graph, so kernels replayed from a CUDA graph are
    timed on the stream that launches them, live, like eager ones (outside a capture it is
    an ordinary record).  Driver API through ctypes (measurement plumbing, not the path)."""
    _cu = None

    def __init__(self):
        import ctypes
        if DrvTimer._cu is None:
            cu = ctypes.CDLL("libcuda.so.1")
            cu.cuEventCreate.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_uint]
            cu.cuEventRecordWithFlags.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
            cu.cuEventElapsedTime.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_void_p,
                                              ctypes.c_void_p]
            cu.cuEventDestroy_v2.argtypes = [ctypes.c_void_p]
            cu.cuStreamIsCapturing.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
            DrvTimer._cu = cu
        self.ev = ctypes.c_void_p()
        torch.cuda.current_stream()   # the primary context is current on this thread
        r = DrvTimer._cu.cuEventCreate(ctypes.byref(self.ev), 0)
        if r != 0:
            raise RuntimeError(f"cuEventCreate: {r}")

    def record(self, stream=None):
        import ctypes
        s = torch.cuda.current_stream() if stream is None else stream
        st = ctypes.c_int(0)   # the EXTERNAL flag is only valid while the stream captures
        DrvTimer._cu.cuStreamIsCapturing(s.cuda_stream, ctypes.byref(st))
        r = DrvTimer._cu.cuEventRecordWithFlags(self.ev, s.cuda_stream, 1 if st.value == 1 else 0)
        if r != 0:
            raise RuntimeError(f"cuEventRecordWithFlags: {r}")

    def elapsed_time(self, end) -> float:
        """ms between two recorded events; NaN if either was never recorded (e.g. the
        migration timers of a step without hand-off)."""
        import ctypes
        ms = ctypes.c_float()
        r = DrvTimer._cu.cuEventElapsedTime(ctypes.byref(ms), self.ev, end.ev)
        if r != 0:
            return float("nan")
        return float(ms.value)

    def __del__(self):
        try:
            DrvTimer._cu.cuEventDestroy_v2(self.ev)
        except Exception:
            pass


def _capture_steps(step, q, out, lse, K, world, device, timers=None, bounds=None):
    """ONE CUDA graph holding K consecutive steps (every stream, every layer; timers[k] and
    the step boundaries as event-record nodes), captured on every rank; None on every rank
    if any rank could not capture (then the caller runs eagerly)."""
    g, why = None, ""
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(K):
                step.enqueue(q, out, lse, **({} if timers is None else {"timers": timers[k]}))
                if bounds is not None and k < K - 1:
                    bounds[k].record()
    except Exception as e:
        g, why = None, repr(e)[:200]
        log("graph capture failed:", why)
    torch.cuda.synchronize()
    if not _all_true(g is not None, world, device):
        return None, why or "a peer could not capture"
    return g, ""


def run_steps(step, q, out, lse, K, L, world, device, use_graph, timed=True):
    """The timed region of K steps, twice.  Region A (the headline): the K steps with no
    instrumentation -- replayed from ONE CUDA graph per rank (use_graph) or submitted
    eagerly.  Region B (timed=True, right after): the same K steps with per-layer kernel
    events (attention, migration, output-final) as event-record nodes of the graph on the
    launching streams, and step boundaries; the kernel durations (roofline `achieved`)
    come from B.  The events themselves cost ~1-2 % of the step (measured,
    profiles/r02_exp_timers.json), which is why the headline is A.  Returns this rank's ms
    per step of A and B, per-step times and per-layer kernel times of B, host submission
    ms per step, the mode, the clock summary (both regions) and NVLink counters (A)."""
    timers = ([[tuple(DrvTimer() for _ in range(5)) for _ in range(L)] for _ in range(K)]
              if timed else None)
    step_ev = [DrvTimer() for _ in range(K - 1)]
    t0, t1, tb0, tb1 = DrvTimer(), DrvTimer(), DrvTimer(), DrvTimer()
    ga = gb = None
    mode = "eager"
    if use_graph:
        ga, why = _capture_steps(step, q, out, lse, K, world, device)
        if ga is not None and timed:
            gb, why = _capture_steps(step, q, out, lse, K, world, device, timers, step_ev)
        if ga is not None and (gb is not None or not timed):
            mode = "graph"
            for g in (ga, gb):
                if g is not None:
                    g.replay()              # warm each graph (K more untimed steps)
            torch.cuda.synchronize()
            _barrier(world)
            torch.cuda.synchronize()
        else:
            ga = gb = None
            mode = f"eager (graph capture failed: {why})"

    def region(graph, tmr):
        from paper_2510_13223_b200.transport import nvtx
        with nvtx("bench timed region" + (" (instrumented)" if tmr is not None else "")):
            _region(graph, tmr)

    def _region(graph, tmr):
        if graph is not None:
            graph.replay()
            return
        for k in range(K):
            step.enqueue(q, out, lse, **({} if tmr is None else {"timers": tmr[k]}))
            if tmr is not None and k < K - 1:
                step_ev[k].record()
    nvl = NvlinkCounters(device.index) if world > 1 else None
    with ClockSampler(torch.cuda.current_device()) as clk:
        nv0 = nvl.read() if nvl else None
        t0.record()
        h0 = time.perf_counter()
        region(ga, None)
        host_ms = (time.perf_counter() - h0) * 1e3 / K
        t1.record()
        torch.cuda.synchronize()
        nv1 = nvl.read() if nvl else None
        _barrier(world)
        if timed:
            torch.cuda.synchronize()
            tb0.record()
            region(gb, timers)
            tb1.record()
            torch.cuda.synchronize()
    _barrier(world)
    r = {"ms": t0.elapsed_time(t1) / K, "mode": mode, "host_ms": host_ms, "clocks": clk.summary(),
         "nvlink": NvlinkCounters.delta(nv0, nv1, K) if world > 1 else None}
    if timed:
        bounds = [tb0] + step_ev + [tb1]
        r["ms_instrumented"] = tb0.elapsed_time(tb1) / K
        r["per_step"] = sorted(a.elapsed_time(b) for a, b in zip(bounds[:-1], bounds[1:]))
        r["attn_ms"] = [t[0].elapsed_time(t[1]) for tk in timers for t in tk]
        r["mig_ms"] = [t[2].elapsed_time(t[3]) for tk in timers for t in tk]
        # attention end -> out[l] final: the exchange + merge latency after the launch
        r["out_ms"] = [t[1].elapsed_time(t[4]) for tk in timers for t in tk]
    del ga, gb
    return r


def _same_gpu() -> bool:
    return os.environ.get("BS_RING_SAME_GPU", "0") == "1"


# --------------------------------------------------------------------------------------
# C2: the home/cold ring (headline)
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
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32).to(device)  # noqa: E731
    step = ShardedDecodeStep(
        CudaOps(synth.default_scale(SHAPE.d)), CudaExec(device), rank, world, home, i32(home_bt),
        cold, i32(cold_bt), i32(ks), SHAPE.hq, L, SHAPE.d, handoff_src_ids=i32(src_ids),
        handoff_dst_ids=i32(dst_ids), chunk_bytes=home.chunk_bytes,
        pg_attn=dist.group.WORLD if world > 1 else None,
        pg_mig=dist.new_group(list(range(world))) if world > 1 else None,
        lookahead=int(os.environ.get("BS_LOOKAHEAD", "-1")), device=device,
        copy_engine=os.environ.get("BS_HANDOFF_CE", "0") == "1",
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


def _e2e_buffers(q, extra, L, device):
    """Pinned host rows + device rows [q_l | extra_l] per layer (one H2D copy per layer)."""
    qb = q[0].numel() * q.element_size()
    kvb = 0 if extra is None else extra[0].numel() * extra.element_size()
    rowb = qb + kvb
    in_host = torch.empty((L, rowb), dtype=torch.uint8).pin_memory()
    in_dev = torch.empty((L, rowb), dtype=torch.uint8, device=device)
    in_host[:, :qb].copy_(q.cpu().view(torch.uint8).reshape(L, qb))
    q_dev = in_dev[:, :qb].view(q.dtype).view(q.shape)
    extra_dev = None
    if extra is not None:
        in_host[:, qb:].copy_(extra.cpu().view(torch.uint8).reshape(L, kvb))
        extra_dev = in_dev[:, qb:].view(extra.dtype).view(extra.shape)
    return in_host, in_dev, rowb, q_dev, extra_dev


def e2e_measure(bs, step, q_dev, out, lse, in_host, in_dev, rowb, out_host, lse_host, L, K,
                world, device, use_graph):
    """K end-to-end steps: per layer one H2D copy of [q_l | extra_l] from pinned memory (a
    side stream; layer l's attention waits only for its own inputs), the step, per layer
    the D2H copies of O_l / lse_l as each layer lands, and the host waiting for the result
    every step -- every copy through the library's bs_copy_bytes (C-ABI).  One such step is
    one CUDA graph replayed per step when possible.  Returns (ms per step, mode)."""
    h2d = torch.cuda.Stream(device=device)
    d2h = torch.cuda.Stream(device=device)
    q_ev = [torch.cuda.Event() for _ in range(L)]
    ob, lb = out[0].numel() * out.element_size(), lse[0].numel() * lse.element_size()

    def one():
        cur = torch.cuda.current_stream()
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

    g, mode = None, "eager"
    if use_graph:
        one()
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                one()
        except Exception as e:
            g = None
            mode = f"eager (graph capture failed: {repr(e)[:120]})"
        torch.cuda.synchronize()
        if not _all_true(g is not None, world, device):
            g = None
        elif g is not None:
            mode = "graph (one CUDA graph per e2e step: H2D copies + step + D2H copies)"

    def e2e_step():
        if g is not None:
            g.replay()
        else:
            one()
        torch.cuda.current_stream().synchronize()  # the next decode step needs the result
    for _ in range(2):
        e2e_step()
    _barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    return _max_over_ranks(e0.elapsed_time(e1) / K, world, device), mode


def run_c2(args, rank, world, device):
    import paper_2510_13223_b200 as bs

    torch.cuda.set_device(device)
    same_gpu = world > 1 and _same_gpu()
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

    h0 = time.perf_counter()
    for _ in range(args.warmup):
        step.enqueue(q, out, lse)
    host_ms = _max_over_ranks((time.perf_counter() - h0) * 1e3 / args.warmup, world, device)
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()

    # ---- timed region: K steps replayed from one CUDA graph per rank (eager with the NCCL
    # transport); kernel events are live graph nodes on their launching streams ----------
    K = args.steps
    use_graph = world == 1 or step.transport == "p2p"
    if step.links is not None:
        step.links.check()
    run = run_steps(step, q, out, lse, K, L, world, device, use_graph)
    if step.links is not None:
        step.links.check()
    ms_max = _max_over_ranks(run["ms"], world, device)
    per_step, attn_ms, mig_ms = run["per_step"], run["attn_ms"], run["mig_ms"]
    # ---- exposure of the migration: the same steps without hand-offs --
    n_handoff, step.n_handoff = step.n_handoff, 0
    for _ in range(2):
        step.enqueue(q, out, lse)
    torch.cuda.synchronize()
    _barrier(world)
    comp = run_steps(step, q, out, lse, K, L, world, device, use_graph, timed=False)
    step.n_handoff = n_handoff
    ms_compute = _max_over_ranks(comp["ms"], world, device)
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
    # ---- the same steps submitted eagerly (host-side cost of the Python protocol) -------
    eager = None
    if run["mode"] == "graph":
        er = run_steps(step, q, out, lse, K, L, world, device, use_graph=False, timed=False)
        eager = {"ms_per_step": round(_max_over_ranks(er["ms"], world, device), 4),
                 "host_submit_ms_per_step": round(_max_over_ranks(er["host_ms"], world, device), 4)}
    if step.links is not None:
        step.links.check()
    clk = run["clocks"]

    # ---- e2e: same step through host buffers ----------------------------------------
    # every step: q copied H2D from pinned memory layer by layer on its own stream (layer
    # l's attention waits only for its own q), O / lse copied D2H layer by layer as each
    # layer finishes, then the host waits for the step's result (the next decode step needs
    # it).  The copies ride the copy engines under the previous/next layers' compute.
    # The step's inputs of layer l -- q_l and (H7) the decoded token's K/V kv_l -- sit
    # packed in one row [q_l | kv_l] of a pinned host buffer and of a device buffer, so each
    # layer is ONE copy; the step reads q and its append K/V as strided views of that buffer.
    # One e2e step (copies + step) is one CUDA graph replayed per decode step when the step
    # itself is graph-capturable, else submitted eagerly.
    kv0 = step.append
    in_host, in_dev, rowb, q_dev, kv_dev = _e2e_buffers(q, kv0, L, device)
    if kv0 is not None:
        step.append = kv_dev
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    lse_host = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
    e2e_ms, e2e_mode = e2e_measure(bs, step, q_dev, out, lse, in_host, in_dev, rowb, out_host,
                                   lse_host, L, K, world, device, use_graph)
    if step.links is not None:
        step.links.check()   # every wait of the e2e steps completed in time
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
    if world == 1:
        fused_app = step.append is not None and step.ce_ids is None
        app_bytes = (2 * step.append[0].numel() * step.append.element_size()) if fused_app else 0
        hbm = 2 * mig_bytes + app_bytes   # hand-off read + write (+ H7 rows read + written)
        rmig = {
            "bound": "hbm",
            "kernel": ("migrate_append_vec16 (hand-off copy + H7 append, one launch on the "
                       "migration stream)" if fused_app else "copy_pages_vec16 (hand-off, copy stream)"),
            "achieved": round(hbm / (mig_avg_ms * 1e-3) / 1e9, 1), "peak": peak,
            "peak_source": peak_src, "unit": "GB/s",
            "frac": round(hbm / (mig_avg_ms * 1e-3) / 1e9 / peak, 4),
            "algorithmic_bytes_per_launch": hbm,
            "note": "read + write bytes; in-step, concurrent with the HBM-bound attention",
            "traffic": ncu_traffic("ncu_copy.json")[0], "traffic_source": ncu_traffic("ncu_copy.json")[1]}
    elif same_gpu:
        rmig = None   # no byte crossed NVLink: the ranks share one GPU
    else:
        rmig = {
            "bound": "nvlink", "kernel": ("copy_pages_vec16 push into the peer's pool"
                                          if step.transport == "p2p" else "gather/NCCL/scatter"),
            "achieved": round(mig_gbs, 1), "peak": NVLINK_GBS_PER_DIR,
            "peak_source": "spec (NVLink 5: 900 GB/s per direction per GPU)", "unit": "GB/s",
            "frac": round(mig_gbs / NVLINK_GBS_PER_DIR, 4),
            "note": "payload per direction per GPU (every rank sends to prev and receives from next)"}
    if not mig_bytes:
        rmig = None
    res = {
        "metric": METRIC,
        "value": round(tokens_s, 2),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max, 4),
        "step_ms_stats": step_stats(per_step),  # instrumented replay (step boundaries)
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 KV/q, Llama-2-7B shape, random-init; no weights)",
        "config": {
            "workload": WORKLOAD, "name": "c2",
            "layers": L, "batch": BATCH, "seq_len": SEQ, "num_q_heads": SHAPE.hq,
            "num_kv_heads": SHAPE.hkv, "head_dim": SHAPE.d, "kv_shards": N_SHARDS,
            "handoff_requests_per_step": N_HANDOFF,
            "h7_append": step.append is not None,
            "parallelism": (f"ring of {world} instances (home + cold per GPU), {step.transport} transport"
                            + (", fused exchange (partials stored into the home GPU's workspace, "
                               "last-arriving CTA merges)" if step.fused_exchange else "")
                            + (f" (p2p unavailable: {step.fallback_reason})"
                               if getattr(step, "fallback_reason", None) else "")
                            + (" [ALL RANKS ON ONE GPU: functional check only]" if same_gpu else "")
                            if world > 1 else "1 GPU, 2 virtual instances"),
            "l2": "no flush: resident pools 70 GiB >> 126 MB L2",
        },
        "attn_hbm_gbs": round(attn_gbs, 1),
        "attn_ms_per_layer": round(attn_avg_ms, 5),
        "migrate_gbs": round(mig_gbs, 1),
        "migrate_ms_per_layer": round(mig_avg_ms, 5),
        "migrate_bytes_per_layer": mig_bytes,
        "exchange_ms_per_layer": round(statistics.fmean(run["out_ms"]), 5),
        "exchange_note": ("mean over layers of attention-launch end -> out[l] final on this rank "
                          "(N>1: the other GPU's partials stored into this GPU's workspace, its "
                          "last-arriver merges and the done-counter wait; N=1: merged in the "
                          "launch, ~0)"),
        "migrate_transport": ("fused copy kernel, local HBM (N=1: both instances on GPU 0)" if world == 1
                              else ("copy kernel pushing into the peer's IPC-mapped pool (P2P, NVLink)"
                                    if step.transport == "p2p" else
                                    "gather -> NCCL send/recv (library bs_comm) -> scatter")
                              + (" [same GPU: no NVLink]" if same_gpu else "")),
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
        # attention beside it), NVLink payload per direction at N>1 on distinct GPUs
        "roofline_migrate": rmig,
        "nvlink_counters": run["nvlink"],
        "overlap": {"step_ms": round(ms_max, 4), "compute_only_ms": round(ms_compute, 4),
                    "exposure": round((ms_max - ms_compute) / ms_compute, 4),
                    "migrate_only_ms": None if ms_mig_only is None else round(ms_mig_only, 4),
                    "overlap_efficiency": (None if ms_mig_only is None else round(
                        (ms_compute + ms_mig_only - ms_max) / min(ms_compute, ms_mig_only), 4)),
                    "migrate_bytes_per_step": mig_bytes * L,
                    "note": ("N=1: the hand-off and the attention share one GPU's HBM, so the "
                             "hand-off's bytes cannot be hidden; over NVLink (N>1) its write side "
                             "leaves the GPU") if world == 1 else "N>1"},
        "timing": {"mode": run["mode"], "compute_only_mode": comp["mode"],
                   "ms_per_step_instrumented": round(_max_over_ranks(run["ms_instrumented"], world,
                                                                     device), 4),
                   "eager": eager, "eager_host_submit_ms_per_step": round(host_ms, 4),
                   "note": "graph: the K timed steps replayed from ONE CUDA graph per rank "
                           "(headline, no instrumentation); the kernel times (roofline) come from "
                           "an instrumented replay of the same K steps right after it (events as "
                           "graph nodes on the launching streams; ms_per_step_instrumented); "
                           "eager = the same K steps submitted from Python; "
                           "eager_host_submit_ms_per_step = the Python/ctypes submission cost of "
                           "one step (warm-up steps, max over ranks)"},
        "gpu_launches": step.launches_per_step * K,
        "e2e": {"value": round(BATCH * world / (e2e_ms * 1e-3), 2), "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 4), "mode": e2e_mode,
                "h2d_bytes_per_step": q.numel() * q.element_size() + (
                    0 if step.append is None else step.append.numel() * step.append.element_size()),
                "d2h_bytes_per_step": out.numel() * out.element_size() + lse.numel() * lse.element_size()},
        "clocks": clk,
    }
    if rank == 0 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(case, budget_s=args.cpu_seconds)
    step.close()
    _barrier(world)
    return res


# --------------------------------------------------------------------------------------
# C3 / C4: W-way sequence sharding, W = number of GPUs
# --------------------------------------------------------------------------------------

SEQ_CONFIGS = {
    "c3": dict(shape=synth.LLAMA3_8B, handoff_tokens=0, scaling="strong",
               workload="C3: Llama-3-8B GQA (L=32, Hq=32, Hkv=8, d=128, bf16 KV), decode B=8 x "
                        "32768 tokens, every request's KV split W ways (W = GPUs; block-aligned), "
                        "request i's home = GPU i mod W merges its W partials (eq. 10)"),
    "c4": dict(shape=synth.LLAMA2_70B, handoff_tokens=8192, scaling="strong",
               workload="C4: Llama-2-70B shape (L=80, Hq=64, Hkv=8, d=128, bf16 KV), decode B=256 "
                        "mixed lengths (50% U{5..40}, 50% log-uniform[2000, 32768], + U{0..511} "
                        "generated; seed 0), every request split W ways, home = i mod W; per layer "
                        "8192 tokens (512 chunks) of KV handed to the next GPU"),
}


def seq_lengths(name):
    if name == "c3":
        return np.full(8, 32768, dtype=np.int64)
    return synth.mixed_lengths(256, seed=0)


def seq_attn_bytes(shape, ks, rank, W):
    """Algorithmic bytes of rank r's launch per layer: range r of every request (KV + block
    table), every home's q (each rank reads all of them) and the merged bf16 O + fp32 lse of
    the requests whose merge it performs (on average B/W of them)."""
    B = ks.shape[0]
    n = (ks[:, rank + 1] - ks[:, rank]).astype(np.int64)
    kv = int(n.sum()) * 2 * shape.hkv * shape.d * 2
    bt = int(sum(4 * synth.ceil_div(int(x), shape.bs) for x in n))
    return kv + bt + B * shape.hq * shape.d * 2 + (B // W) * shape.hq * (shape.d * 2 + 4)


def run_seq(args, rank, world, device, name, headline=False):
    """One W-way sequence-sharded config (W = world) on this rank's GPU."""
    import paper_2510_13223_b200 as bs
    from paper_2510_13223_b200.ring import CudaOps
    from paper_2510_13223_b200.seqshard import SeqShardedStep
    cfg = SEQ_CONFIGS[name]
    shape, W = cfg["shape"], world
    lens = seq_lengths(name)
    B, L = len(lens), shape.n_layers
    if B % W:
        return {"skipped": f"{B} requests do not split over {W} homes"}
    ks = synth.block_aligned_split(lens, W)
    n_hand = cfg["handoff_tokens"] // shape.bs
    my_lens = (ks[:, rank + 1] - ks[:, rank]).astype(np.int64)
    need = (sum(synth.ceil_div(int(x), shape.bs) for x in my_lens) + 2 * n_hand + 1) * L * \
        2 * shape.hkv * shape.bs * shape.d * 2
    free_b = torch.cuda.mem_get_info(device)[0]
    fits = need + (4 << 30) < free_b
    if not _all_true(fits, world, device):
        return {"skipped": f"{name} at W={W}: {need / 1e9:.1f} GB of KV per GPU does not fit "
                           f"({free_b / 1e9:.1f} GB free)"}
    pool_t, bt = synth.device_pool(shape, my_lens, synth.shard_seed(7, rank), device,
                                   spare_blocks=2 * n_hand + 1)
    pool = bs.KVPool(L, pool_t.shape[1], shape.hkv, shape.d, base=pool_t.reshape(-1))
    used = set(int(x) for x in bt.ravel() if x >= 0)
    free = [i for i in range(pool_t.shape[1]) if i not in used]
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32, device=device)  # noqa: E731
    src = i32(free[:n_hand]) if n_hand else None
    dst = i32(free[n_hand:2 * n_hand]) if n_hand else None
    transport = "p2p" if args.transport == "p2p" else "collective"
    step = SeqShardedStep(CudaOps(synth.default_scale(shape.d)), rank, W, pool, i32(bt), i32(ks),
                          shape.hq, L, shape.d, shape.hkv, device=device,
                          group=torch.distributed.group.WORLD if W > 1 else None,
                          transport=transport, handoff_src_ids=src, handoff_dst_ids=dst)
    same_gpu = W > 1 and _same_gpu()
    q = synth.device_q(shape, B, 5, device)[:, rank::W].contiguous()
    own = step.outputs()
    if own is not None:
        out, lse = own
    else:
        out = torch.empty((L, B // W, shape.hq, shape.d), dtype=torch.bfloat16, device=device)
        lse = torch.empty((L, B // W, shape.hq), dtype=torch.float32, device=device)
    p2p = step.transport == "p2p"
    h0 = time.perf_counter()
    for _ in range(args.warmup):
        step.enqueue(q, out, lse)
    host_ms = _max_over_ranks((time.perf_counter() - h0) * 1e3 / args.warmup, world, device)
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    K = args.steps
    run = run_steps(step, q, out, lse, K, L, world, device, use_graph=p2p, timed=p2p)
    step.check()
    ms_max = _max_over_ranks(run["ms"], world, device)
    # compute-only steps (no hand-off) -> exposure of the hand-off
    ms_compute = None
    if n_hand:
        step.n_handoff = 0
        for _ in range(2):
            step.enqueue(q, out, lse)
        torch.cuda.synchronize()
        _barrier(world)
        comp = run_steps(step, q, out, lse, K, L, world, device, use_graph=p2p, timed=False)
        step.n_handoff = n_hand
        ms_compute = _max_over_ranks(comp["ms"], world, device)
    eager = None
    if run["mode"] == "graph":
        er = run_steps(step, q, out, lse, K, L, world, device, use_graph=False, timed=False)
        eager = {"ms_per_step": round(_max_over_ranks(er["ms"], world, device), 4),
                 "host_submit_ms_per_step": round(_max_over_ranks(er["host_ms"], world, device), 4)}
    step.check()
    # e2e through host buffers (P2P transport): q H2D per layer, O / lse D2H per layer
    e2e = None
    if p2p:
        in_host, in_dev, rowb, q_dev, _ = _e2e_buffers(q, None, L, device)
        out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        lse_host = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
        e2e_ms, e2e_mode = e2e_measure(bs, step, q_dev, out, lse, in_host, in_dev, rowb, out_host,
                                       lse_host, L, K, world, device, True)
        step.check()
        e2e = {"value": round(B / (e2e_ms * 1e-3), 2), "unit": "tokens/s",
               "ms_per_step": round(e2e_ms, 4), "mode": e2e_mode,
               "h2d_bytes_per_step": q.numel() * q.element_size(),
               "d2h_bytes_per_step": out.numel() * out.element_size() + lse.numel() * lse.element_size(),
               "note": "per rank: its home requests' q in, their O / lse out; max over ranks"}
    a_bytes = seq_attn_bytes(shape, ks, rank, W)
    peak, peak_src = peaks()
    res = {"metric": METRIC, "value": round(B / (ms_max * 1e-3), 2), "unit": "tokens/s",
           "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
           "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (seeded N(0,1) bf16 KV/q, random-init; no weights)",
           "config": {"workload": cfg["workload"], "name": name, "layers": L, "batch": B,
                      "context_tokens": int(lens.sum()), "kv_shards": W,
                      "num_q_heads": shape.hq, "num_kv_heads": shape.hkv, "head_dim": shape.d,
                      "handoff_tokens_per_layer": cfg["handoff_tokens"],
                      "parallelism": (f"{W}-way sequence sharding, {step.transport} transport"
                                      + (", fused exchange (partials into each home's workspace, "
                                         "last-arriving CTA merges)" if p2p else "")
                                      + (" [ALL RANKS ON ONE GPU: functional check only]"
                                         if same_gpu else "")),
                      "l2": "no flush: every step reads >= 4 GiB of distinct KV per GPU >> 126 MB L2"},
           "timing": {"mode": run["mode"], "eager": eager,
                      "ms_per_step_instrumented": (round(_max_over_ranks(
                          run["ms_instrumented"], world, device), 4) if p2p else None),
                      "eager_host_submit_ms_per_step": round(host_ms, 4)},
           "gpu_launches": step.launches_per_step * K, "e2e": e2e, "clocks": run["clocks"],
           "nvlink_counters": run["nvlink"]}
    if p2p:
        attn_avg = statistics.fmean(run["attn_ms"])
        gbs = a_bytes / (attn_avg * 1e-3) / 1e9
        res["attn_hbm_gbs_per_gpu"] = round(gbs, 1)
        res["attn_ms_per_layer"] = round(attn_avg, 5)
        res["roofline"] = {"bound": "hbm", "kernel": "split_decode_attn_mma via "
                           "bs_split_decode_attention_tasks (range r of every home's requests)",
                           "achieved": round(gbs, 1), "peak": peak, "peak_source": peak_src,
                           "unit": "GB/s", "frac": round(gbs / peak, 4), "traffic": None,
                           "algorithmic_bytes_per_layer": a_bytes, "rank": rank}
        # attention end -> out[l] final on this rank: the peers' partial stores into this
        # rank's homes' workspaces, their last-arriver merges and the done wait
        res["exchange_ms_per_layer"] = round(statistics.fmean(run["out_ms"]), 5)
        if n_hand:
            mig_avg = statistics.fmean(run["mig_ms"])
            mb = n_hand * pool.chunk_bytes
            res["migrate_bytes_per_layer"] = mb
            res["migrate_gbs"] = round(mb / (mig_avg * 1e-3) / 1e9, 1)
            res["roofline_migrate"] = None if (W == 1 or same_gpu) else {
                "bound": "nvlink", "kernel": "copy_pages_vec16 push into the next GPU's pool",
                "achieved": res["migrate_gbs"], "peak": NVLINK_GBS_PER_DIR,
                "peak_source": "spec (NVLink 5: 900 GB/s per direction per GPU)", "unit": "GB/s",
                "frac": round(res["migrate_gbs"] / NVLINK_GBS_PER_DIR, 4)}
    if ms_compute is not None:
        res["overlap"] = {"step_ms": round(ms_max, 4), "compute_only_ms": round(ms_compute, 4),
                          "exposure": round((ms_max - ms_compute) / ms_compute, 4),
                          "migrate_bytes_per_step": n_hand * pool.chunk_bytes * L}
    if headline and rank == 0 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_seq(name, budget_s=args.cpu_seconds)
    step.close()
    _barrier(world)
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
                       f"{N_HANDOFF} hand-offs, {SHAPE.n_layers} layers (one GPU's share)"),
            "measured_seconds": round(ta_tot + tm_tot, 3)}


class SeqOracleSample:
    """A bounded host sample of a sequence-sharded config for the oracle: a few seeded
    requests of one layer with their KV in W shard pools (the config's split), plus the
    hand-off chunks of one layer; extrapolated to the full step by context tokens."""

    def __init__(self, name, W, n_req=2):
        cfg = SEQ_CONFIGS[name]
        self.shape, self.name, self.W = cfg["shape"], name, W
        self.lens_all = seq_lengths(name)
        # the requests at the 50th and 90th length percentiles (mixed-length batches: the
        # long ones carry most of the work the extrapolation scales to)
        order = np.argsort(self.lens_all, kind="stable")
        qs = np.linspace(0.5, 0.9, n_req) if n_req > 1 else np.array([0.5])
        pick = np.sort(order[(qs * (len(order) - 1)).round().astype(int)])
        lens = self.lens_all[pick]
        ks = synth.block_aligned_split(lens, W)
        one = synth.Shape(1, self.shape.hq, self.shape.hkv, self.shape.d)
        case = synth.device_shards(one, lens, ks, seed=31, device="cpu", layers=1)
        self.sample = synth.extract_requests(case, list(range(n_req)), 0)
        self.tokens = int(lens.sum())
        self.n_hand = cfg["handoff_tokens"] // self.shape.bs
        cb = 2 * self.shape.hkv * self.shape.bs * self.shape.d
        self.src = np.zeros((1, max(self.n_hand, 1), cb), dtype=np.uint16) if self.n_hand else None
        self.scale = synth.default_scale(self.shape.d)

    def time_once(self):
        import oracle
        sp, sbt, sks, sq = self.sample
        t = time.perf_counter()
        parts = [oracle.attention_shard(p, 0, sq, bt, sks, j, self.scale)
                 for j, (p, bt) in enumerate(zip(sp, sbt))]
        oracle.merge_partials([x[0] for x in parts], [x[1] for x in parts], [x[2] for x in parts])
        ta = time.perf_counter() - t
        tm = 0.0
        if self.src is not None:
            src = self.src.reshape(1, self.n_hand, 2, self.shape.hkv, self.shape.bs, self.shape.d)
            dst = np.empty_like(src)
            t = time.perf_counter()
            oracle.migrate_layer(src, dst, 0, np.arange(self.n_hand), np.arange(self.n_hand))
            tm = time.perf_counter() - t
        return ta, tm

    def step_seconds(self, ta, tm):
        """Full step: L layers x (all requests' attention scaled by context tokens + each
        rank's hand-off chunks)."""
        scale_tokens = float(self.lens_all.sum()) / self.tokens
        return self.shape.n_layers * (ta * scale_tokens + tm * self.W)

    def describe(self, units):
        return (f"{units} timed units of 1 layer x {len(self.sample[3])} requests ({self.tokens} "
                f"context tokens, all {self.W} shards + LSE merge"
                + (f", + {self.n_hand} hand-off chunks" if self.n_hand else "")
                + f"), fp64 C oracle; extrapolated by context tokens to all {len(self.lens_all)} "
                f"requests and {self.shape.n_layers} layers")


def cpu_baseline_seq(name, budget_s=12.0):
    import oracle
    oracle.lib()
    W = max(1, int(os.environ.get("WORLD_SIZE", "1")))
    smp = SeqOracleSample(name, W)
    ta_tot = tm_tot = 0.0
    units = 0
    while units < 200 and ta_tot + tm_tot < budget_s:
        ta, tm = smp.time_once()
        ta_tot += ta
        tm_tot += tm
        units += 1
    t_step = smp.step_seconds(ta_tot / units, tm_tot / units)
    B = len(smp.lens_all)
    return {"value": round(B / t_step, 4), "unit": "tokens/s", "kind": "oracle", "cores": omp_threads(),
            "nproc": os.cpu_count(), "cpu_model": cpu_model(), "sample": smp.describe(units),
            "measured_seconds": round(ta_tot + tm_tot, 3)}


def run_reference(args, rank, world, device):
    """--impl reference: the CPU oracle as the reference arm, per step a bounded sample of
    the same workload.  `ms_per_step` is the MEASURED time of one timed step (one sample);
    `value` extrapolates that sample to the full step (stated in `extrapolation`)."""
    import oracle

    oracle.lib()
    cores = omp_threads()
    name = "c2" if args.config in ("auto", "c2") else args.config
    if name == "c2":
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
        one = lambda i: time_oracle_sample(samples[i % 2], scale)  # noqa: E731
        full = lambda ta, tm: SHAPE.n_layers * (ta * BATCH / reqs + tm * N_HANDOFF)  # noqa: E731
        B, workload = BATCH * world, WORKLOAD
        sample = (f"per step: 1 layer x {reqs} requests (H7 append + both shards + merge) + 1 "
                  f"hand-off request's chunks, fp64 C oracle")
        extrap = (f"x {BATCH // reqs} requests x {N_HANDOFF} hand-offs x {SHAPE.n_layers} layers "
                  f"(x {world} GPUs' shares, serially)")
        full_b = lambda ta, tm: full(ta, tm) * world  # noqa: E731
    else:
        smp = SeqOracleSample(name, world)
        one = lambda i: smp.time_once()  # noqa: E731
        full_b = smp.step_seconds
        B, workload = len(smp.lens_all), SEQ_CONFIGS[name]["workload"]
        sample = "per step: " + smp.describe(1)
        extrap = "by context tokens to the whole batch and all layers"
    for i in range(args.warmup):
        one(i)
    ta = tm = 0.0
    t0 = time.perf_counter()
    for i in range(args.steps):
        a, m = one(i)
        ta += a
        tm += m
    wall = time.perf_counter() - t0
    t_full = full_b(ta / args.steps, tm / args.steps)
    v = B / t_full
    return {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(wall / args.steps * 1e3, 3),
            "extrapolation": {"full_step_ms": round(t_full * 1e3, 3), "how": extrap,
                              "note": "value = requests / full_step_ms (extrapolated from the "
                                      "measured sample); ms_per_step is the measured sample time"},
            "higher_is_better": True, "scaling": "weak" if name == "c2" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "name": name, "parallelism": "CPU oracle"},
            "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "kind": "oracle",
                             "cores": cores, "sample": sample},
            "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "measured_seconds": round(wall, 3)}


# --------------------------------------------------------------------------------------
# launch
# --------------------------------------------------------------------------------------

def run_shares(device) -> dict:
    """N=1 only: the C4 and C5 per-GPU steps at one GPU's share of 8 (scripts/bench_c4.py,
    bench_c5.py) -- the KV a GPU of the 8-GPU configs holds, the hand-off / prefix migration
    it receives coming from a second pool in local HBM (HBM-bound here; NVLink at 8 GPUs).
    Eager submission, CUDA events, 3 warm-up + 10 timed steps, pools >> L2."""
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    out = {}
    for name in ("c4_share", "c5_share"):
        _release(1)
        try:
            if name == "c4_share":
                import bench_c4
                r = bench_c4.run(device=device)
                v = r["decode_tokens_per_s_per_gpu_share"]
            else:
                import bench_c5
                r = bench_c5.run(device=device)
                v = r["decode_tokens_per_s"]
            out[name] = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": 1,
                         "scaling": "one GPU's share of an 8-GPU config", "dtype": "bf16",
                         "data": "synthetic", "higher_is_better": True,
                         "note": ("one GPU's share of BASELINE config " + ("C4" if name == "c4_share" else "C5")
                                  + "; the migrated KV comes from a second pool in this GPU's HBM "
                                  "(HBM-bound here, NVLink-bound at 8 GPUs)"), **r}
        except Exception as e:  # report, keep the headline line
            out[name] = {"error": repr(e)[:300]}
            log(f"extra config {name} failed:", repr(e))
    _release(1)
    return out


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(n: int) -> int:
    """`--gpus N` (N > 1) outside torchrun: re-run this script under torch.distributed.run,
    one rank per GPU; rank 0 prints the JSON line.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    log("bench.py: launching", n, "ranks:", " ".join(cmd))
    return subprocess.call(cmd)


def fail(msg: str, code: int = 2):
    print(json.dumps({"metric": METRIC, "error": msg}), flush=True)
    log("bench.py: error:", msg)
    sys.exit(code)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["auto", "c2", "c3", "c4"], default="auto",
                    help="auto: C2 headline + C3 (and C4 at N>=4) under extra_configs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-share-configs", action="store_true",
                    help="N=1: skip the C4 / C5 one-GPU-share steps under extra_configs")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--transport", choices=["p2p", "nccl"], default=os.environ.get("BS_TRANSPORT", "p2p"),
                    help="N>1 exchange: CUDA-IPC pushes + flags (p2p) or the library's NCCL "
                         "communicator (nccl)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "ours" and not _same_gpu() and torch.cuda.device_count() < args.gpus:
            fail(f"--gpus {args.gpus} but only {torch.cuda.device_count()} GPU(s) visible "
                 "(BS_RING_SAME_GPU=1 runs every rank on cuda:0 as a functional check)")
        sys.exit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        fail(f"WORLD_SIZE={world} but --gpus {args.gpus}: launch one rank per GPU")
    same_gpu = _same_gpu()
    if args.impl == "reference":  # rank 0 alone runs it; other ranks exit without work
        device = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
        if rank == 0:
            print(json.dumps(run_reference(args, rank, world, device)), flush=True)
        return
    if world > 1 and not same_gpu and torch.cuda.device_count() < world:
        fail(f"{world} ranks but {torch.cuda.device_count()} GPU(s) visible")
    # functional check of the N>1 path on a 1-GPU box: every rank on cuda:0 (time-sliced,
    # numbers meaningless), gloo for the host plumbing, P2P transport
    device = torch.device("cuda", 0 if same_gpu else local)
    torch.cuda.set_device(device)
    if world > 1:
        if same_gpu:
            args.transport = "p2p"
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=device)
    try:
        head = "c2" if args.config == "auto" else args.config
        if head == "c2":
            res = run_c2(args, rank, world, device)
        else:
            res = run_seq(args, rank, world, device, head, headline=True)
            if "skipped" in res:
                fail(res["skipped"])
        if args.config == "auto":
            extras = {}
            for name in ("c3", "c4"):
                if name == "c4" and world < 4:
                    extras[name] = {"skipped": "C4's 457-533 GB of KV needs >= 4 GPUs"}
                    continue
                _release(world)
                try:
                    extras[name] = run_seq(args, rank, world, device, name)
                except Exception as e:  # report, keep the headline line
                    extras[name] = {"error": repr(e)[:300]}
                    log(f"extra config {name} failed:", repr(e))
            if world == 1 and not args.no_share_configs:
                extras.update(run_shares(device))
            res["extra_configs"] = extras
        if rank == 0:
            print(json.dumps(res), flush=True)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
