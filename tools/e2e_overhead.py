#!/usr/bin/env python
"""Where the host-side microseconds of one individual go: device time, mmx_measure from Python one call at a time, the same
individuals through one mmx_measure_batch call (no Python between them).  python tools/e2e_overhead.py [N]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
G = "101010101001"
K = 2000
with capi.Context(n=n, timeout_s=600.0) as ctx:
    for _ in range(20):
        ctx.measure(G)
    t0 = time.perf_counter()
    dev = 0.0
    for _ in range(K):
        dev += ctx.measure(G).time_s
    wall = time.perf_counter() - t0
    t0 = time.perf_counter()
    outs = ctx.measure_batch([G] * K)
    wall_b = time.perf_counter() - t0
    dev_b = sum(o.time_s for o in outs)
    t0 = time.perf_counter()
    for _ in range(K):
        capi.genome_bits(G)
    bits = time.perf_counter() - t0
    print(json.dumps({"n": n, "device_us": dev / K * 1e6, "python_call_wall_us": wall / K * 1e6, "batch_wall_us": wall_b / K * 1e6,
                      "batch_device_us": dev_b / K * 1e6, "genome_bits_us": bits / K * 1e6}))
