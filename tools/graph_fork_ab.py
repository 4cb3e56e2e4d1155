#!/usr/bin/env python
"""A/B of the forked whole-individual graph: MMX_GRAPH_FORK=1 (default: init-a and zero-c on side lanes beside init-b -> transpose)
against =0 (one chain).  python tools/graph_fork_ab.py [N ...]"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import json, sys
sys.path.insert(0, %r)
from paper_1806_01430_b200 import capi
n, dtype = int(sys.argv[1]), int(sys.argv[2])
with capi.Context(n=n, dtype=dtype, timeout_s=600.0) as ctx:
    for _ in range(5):
        ctx.measure("101010101001")
    ts = sorted(ctx.measure("101010101001").time_s for _ in range(100))
    print(json.dumps({"n": n, "dtype": "f64" if dtype == 0 else "f32", "median_ms": ts[len(ts) // 2] * 1e3, "min_ms": ts[0] * 1e3,
                      "checksum": ctx.stats().checksum}))
''' % str(ROOT)

for n in [int(x) for x in sys.argv[1:]] or [256, 1024, 4096, 8192]:
    for dtype in (0, 1):
        for fork in ("1", "0"):
            env = dict(os.environ, MMX_GRAPH_FORK=fork)
            out = subprocess.run([sys.executable, "-c", CHILD, str(n), str(dtype)], capture_output=True, text=True, env=env)
            row = json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else {"error": out.stderr[-500:]}
            row["graph_fork"] = fork
            print(json.dumps(row), flush=True)
