#!/usr/bin/env python
"""Per-SM read ceiling (diagnostics, see sm_read.cu): one CTA per SM streams 8 MiB of its
own; GB/s per CTA and in total for 16..148 CTAs, LDG (U loads in flight per thread, 512
threads) vs TMA bulk (a ring of S 8-KiB slots).  python scripts/diag/sm_read.py [--json f]"""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libsm_read.so")


def build():
    src = os.path.join(HERE, "sm_read.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", src, "-o", SO])
    return ctypes.CDLL(SO)


def main():
    L = build()
    L.sm_read.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                          ctypes.c_void_p, ctypes.c_void_p]
    per = 8 << 20
    buf = torch.ones(148 * per // 2, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    res = []
    for nctas in (16, 32, 64, 128, 148):
        for mode, param in ((0, 8), (0, 16), (1, 8), (1, 16), (1, 24)):
            ts = []
            for _ in range(5):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                assert L.sm_read(buf.data_ptr(), per, nctas, mode, param, sink.data_ptr(), s) == 0
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            t = sorted(ts)[len(ts) // 2] * 1e-3
            r = {"ctas": nctas, "path": "ldg" if mode == 0 else "tma_bulk",
                 ("loads_in_flight_per_thread" if mode == 0 else "stages_8KiB"): param,
                 "in_flight_KiB_per_cta": (512 * param * 16 if mode == 0 else param * 8192) // 1024,
                 "us": round(t * 1e6, 1), "GBps_per_cta": round(per / t / 1e9, 1),
                 "GBps_total": round(per * nctas / t / 1e9, 1)}
            print(json.dumps(r), flush=True)
            res.append(r)
    if len(sys.argv) > 2 and sys.argv[1] == "--json":
        with open(sys.argv[2], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
