#!/usr/bin/env python
"""NEXT F4 measurement: host latency of the C++ control plane behind the C-ABI.

    python scripts/bench_policy.py [--json out.json]

Alg. 2 (bs_dispatch_requests): a C5-sized burst (512 requests) and a 10k-request queue
over 8 / 64 prefill instances; Alg. 1 (bs_plan_migrations): one control cycle over 8 / 64
devices with random loads (every device supports both move kinds).  Reported: µs per call
(median of repeated calls, time.perf_counter around the ctypes call, arrays prepared
outside the timed region) and the number of moves planned."""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_13223_b200 as bs  # noqa: E402


def median_us(fn, reps):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    t.sort()
    return t[len(t) // 2] * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    args = ap.parse_args()
    L = bs.lib()
    rng = np.random.default_rng(0)
    res = []
    for n_inst, n_req in ((8, 512), (8, 10_000), (64, 10_000)):
        load0 = rng.uniform(0.1, 0.9, n_inst)
        est = rng.uniform(0.001, 0.01, n_req)
        q0 = rng.integers(0, 8, n_inst).astype(np.int32)
        out = np.zeros(n_req, dtype=np.int32)
        ld, ql = load0.copy(), q0.copy()

        def call():
            ld[:] = load0
            ql[:] = q0
            assert L.bs_dispatch_requests(n_inst, ld.ctypes.data, ql.ctypes.data, n_req,
                                          est.ctypes.data, 0.8, out.ctypes.data) == 0
        us = median_us(call, 50)
        r = {"case": f"alg2_dispatch_{n_req}req_{n_inst}inst", "us": round(us, 1),
             "ns_per_request": round(us * 1e3 / n_req, 1)}
        print(json.dumps(r), flush=True)
        res.append(r)
    for n_dev in (8, 64):
        load0 = rng.uniform(0.0, 1.0, n_dev)
        nl0 = np.full(n_dev, 4, dtype=np.int32)
        nh0 = np.full(n_dev, 8, dtype=np.int32)
        ll = np.full(n_dev, 0.05)
        lc = np.full(n_dev, 0.02)
        hl = np.full(n_dev, 0.01)
        hc = np.full(n_dev, 0.002)
        sl = np.ones(n_dev, dtype=np.uint8)
        sa = np.ones(n_dev, dtype=np.uint8)
        mv = np.zeros(3 * 10_000, dtype=np.int32)
        n = ctypes.c_int32()
        ld, nl, nh = load0.copy(), nl0.copy(), nh0.copy()

        def call():
            ld[:] = load0
            nl[:] = nl0
            nh[:] = nh0
            assert L.bs_plan_migrations(n_dev, ld.ctypes.data, nl.ctypes.data, ll.ctypes.data,
                                        lc.ctypes.data, nh.ctypes.data, hl.ctypes.data,
                                        hc.ctypes.data, sl.ctypes.data, sa.ctypes.data, 0.1, 0.5,
                                        10_000, mv.ctypes.data, ctypes.byref(n)) == 0
        us = median_us(call, 50)
        r = {"case": f"alg1_cycle_{n_dev}dev", "us": round(us, 1), "moves": int(n.value),
             "load_spread_before": round(float(load0.max() - load0.min()), 3),
             "load_spread_after": round(float(ld.max() - ld.min()), 3)}
        print(json.dumps(r), flush=True)
        res.append(r)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
