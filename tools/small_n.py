#!/usr/bin/env python
"""Steady-state time of whole individuals at the fixture size (N=256): launch-latency regime."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import cpu  # noqa: E402  (CPU time beside it)
from paper_1806_01430_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for batching in (1, 0):
    with capi.Context(n=n, repetitions=21, warmup=3, launch_batching=batching) as ctx:
        for g in ("101010101001", "100000000000", "000000001000", "101010101000", "010101010101"):
            out = ctx.measure(g)
            t0 = time.perf_counter()
            for _ in range(20):
                ctx.measure(g)
            call_us = (time.perf_counter() - t0) / 20 / 24 * 1e6
            print(json.dumps({"n": n, "batching": batching, "genome": g, "status": out.status, "median_us": round(out.time_s * 1e6, 2),
                              "host_us_per_run": round(call_us, 2)}), flush=True)
r = cpu.time_app(n, 0, 1, n)
print(json.dumps({"cpu_single_thread_us": round(sum(r["seconds"].values()) * 1e6, 1)}))
