#!/usr/bin/env python
"""Pure-read HBM bandwidth (diagnostics): best of 10 per (CTAs/SM, loads in flight) over a
4 GiB buffer, CUDA events.  python scripts/diag/hbm_read.py [--json out.json]"""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libhbm_read.so")


def build():
    src = os.path.join(HERE, "hbm_read.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", src, "-o", SO])
    return ctypes.CDLL(SO)


def main():
    L = build()
    L.hbm_read.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p]
    nbytes = 4 << 30
    buf = torch.ones(nbytes // 2, dtype=torch.bfloat16, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    res = []
    for cps in (1, 2, 4):
        for u in (4, 8, 16):
            ts = []
            for _ in range(12):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                assert L.hbm_read(buf.data_ptr(), nbytes, cps, u, sink.data_ptr(), s) == 0
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            best = min(ts[2:])
            r = {"ctas_per_sm": cps, "threads": 512, "loads_in_flight": u, "GBps": round(nbytes / best / 1e6, 1)}
            print(json.dumps(r), flush=True)
            res.append(r)
    out = {"what": "pure-read HBM bandwidth, 4 GiB, 16-B ld.global.nc, best of 10", "cases": res,
           "max_GBps": max(r["GBps"] for r in res)}
    print(json.dumps({"max_GBps": out["max_GBps"]}))
    if len(sys.argv) > 2 and sys.argv[1] == "--json":
        with open(sys.argv[2], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
