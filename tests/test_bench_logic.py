"""Host-side logic of bench.py (no GPU): algorithmic-byte accounting, hand-off id choice,
clock-log parsing, and the CLI."""
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def test_attention_bytes_closed_form():
    ks = synth.block_aligned_split(np.full(64, 2048), 2)
    hq, d, hkv = 32, 128, 32
    kv = 64 * 2048 * 2 * hkv * d * 2
    bt = 64 * 2 * 4 * 64
    fused = kv + bt + 64 * hq * d * 2 + 64 * hq * (d * 2 + 4)
    split = kv + bt + 64 * hq * d * 2 + 64 * 2 * hq * (d + 2) * 4
    assert bench.attn_bytes_per_layer(ks, fused=True) == fused
    assert bench.attn_bytes_per_layer(ks, fused=False) == split
    assert fused == 2148573184                      # the number bench.py reports per layer


def test_handoff_src_ids_are_lowest_unused_of_the_cold_pool():
    lens = np.array([40, 33])
    ks = synth.block_aligned_split(lens, 2)
    case = synth.device_shards(synth.Shape(1, 2, 2, 64), lens, ks, seed=3, device="cpu",
                               spare_blocks=4, layers=1)
    used = set(int(x) for x in case.block_tables[1].ravel() if x >= 0)
    got = bench.handoff_src_ids(case, 3)
    assert got == sorted(i for i in range(case.pools[1].shape[1]) if i not in used)[:3]
    assert not (set(got) & used)


def test_clock_summary_parsing(tmp_path):
    c = bench.ClockSampler(0)

    class _P:
        pass
    c.proc = _P()
    f = open(tmp_path / "c.csv", "w+")
    f.write("1965, 1965, Not Active, Not Active, Not Active, Active\n"
            "1900, 1965, Not Active, Not Active, Not Active, Not Active\n"
            "garbage line\n")
    f.flush()
    c.f = f
    s = c.summary()
    assert s["sm_mhz"] == 1932.5 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 2


def test_cli_help():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "--transport" in r.stdout and "--impl" in r.stdout


def test_step_stats():
    s = bench.step_stats([1.0, 2.0, 3.0, 4.0])
    assert s["median"] == 2.5 and s["min"] == 1.0 and s["max"] == 4.0 and s["mean"] == 2.5
    assert abs(s["ci95"] - 1.96 * (5 / 3) ** 0.5 / 2) < 1e-4 and s["n"] == 4
    assert bench.step_stats([]) is None


def test_clock_summary_keeps_samples_under_load(tmp_path):
    c = bench.ClockSampler(0)

    class _P:
        pass
    c.proc = _P()
    f = open(tmp_path / "c.csv", "w+")
    f.write("345, 1965, Not Active, Not Active, Not Active, Not Active, 0\n"       # idle
            "1965, 1965, Not Active, Not Active, Not Active, Active, 100\n"
            "1950, 1965, Not Active, Not Active, Not Active, Not Active, 98\n")
    f.flush()
    c.f = f
    s = c.summary()
    assert s["sm_mhz"] == 1957.5 and s["samples"] == 2 and s["reasons"] == ["sw_power_cap"]


def test_clock_summary_nvml_rows():
    """NVML samples (polled inside the timed region only) are all kept."""
    c = bench.ClockSampler(0)
    c.nvml = object()
    c.rows = [(1965.0, 1965.0, 100.0, ["Not Active"] * 4),
              (1800.0, 1965.0, 100.0, ["Not Active", "Not Active", "Not Active", "Active"]),
              (1900.0, 1965.0, 100.0, ["Not Active"] * 4)]
    s = c.summary()
    assert s["sm_mhz"] == 1900.0 and s["sm_mhz_min"] == 1800.0 and s["samples"] == 3
    assert s["reasons"] == ["sw_power_cap"] and s["source"].startswith("nvml")


def test_gpus_flag_fails_loudly_without_enough_gpus():
    """`--gpus N` outside torchrun self-launches N ranks -- unless fewer GPUs are visible:
    then it fails (exit 2, an "error" JSON line) instead of silently measuring N=1."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2
    assert "error" in r.stdout and "GPU" in r.stdout


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stdout


def test_seq_attention_bytes_closed_form():
    """C3 at W=4: rank r reads range r (8192 tokens) of all 8 requests, every home's q, and
    writes the merged O + lse of 2 requests."""
    shape = synth.LLAMA3_8B
    ks = synth.block_aligned_split(np.full(8, 32768), 4)
    kv = 8 * 8192 * 2 * 8 * 128 * 2
    bt = 8 * 4 * 512
    q = 8 * 32 * 128 * 2
    o = 2 * 32 * (128 * 2 + 4)
    for r in range(4):
        assert bench.seq_attn_bytes(shape, ks, r, 4) == kv + bt + q + o


def test_seq_oracle_sample_is_bounded_and_scales_by_tokens():
    smp = bench.SeqOracleSample("c4", 8)
    lens = bench.seq_lengths("c4")
    assert len(lens) == 256 and smp.tokens < lens.sum() // 4
    assert smp.n_hand == 512
    # extrapolation: L x (t_attn x total/sampled tokens + t_mig x W)
    assert abs(smp.step_seconds(1.0, 0.5) - 80 * (lens.sum() / smp.tokens + 0.5 * 8)) < 1e-6


def test_clock_summary_reports_board_power():
    """NVML rows + power samples: the clocks object carries board power (median / max) and
    the enforced limit -- the context of a sw_power_cap run."""
    c = bench.ClockSampler(0)
    c.nvml = object()   # summary() only reads the rows
    c.rows = [(1900.0, 1965.0, 100.0, ["Not Active"] * 3 + ["Active"])] * 4
    c.power = [800.0, 850.0, 910.0, 820.0]
    c.power_limit_w = 1000.0
    s = c.summary()
    assert s["power_w_median"] == 835.0 and s["power_w_max"] == 910.0 and s["power_limit_w"] == 1000.0
    assert s["reasons"] == ["sw_power_cap"]


def test_staged_store_runs():
    """The staged host-tier engine issues one copy-engine transfer per run of consecutive
    store ids, each landing at its pairs' position in the staging buffer."""
    from paper_2510_13223_b200.kvstore import _runs
    assert _runs([]) == []
    assert _runs([7]) == [(7, 1, 0)]
    assert _runs([3, 4, 5, 9, 10, 2]) == [(3, 3, 0), (9, 2, 3), (2, 1, 5)]
    assert _runs(range(100, 164)) == [(100, 64, 0)]
    assert sum(c for _, c, _ in _runs([5, 6, 1, 2, 3, 8])) == 6
