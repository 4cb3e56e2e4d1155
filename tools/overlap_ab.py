#!/usr/bin/env python
"""A/B of the executor's hoisting + streaming around CPU-mapped nests (MMX_OVERLAP=1 default, =0 off) on mixed genomes.
python tools/overlap_ab.py [N]"""
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
n = int(sys.argv[1])
with capi.Context(n=n, timeout_s=600.0) as ctx:
    for genome in sys.argv[2:]:
        ctx.measure(genome)
        ts = sorted(ctx.measure(genome).time_s for _ in range(5))
        st = ctx.stats()
        print(json.dumps({"n": n, "genome": genome, "median_ms": ts[2] * 1e3, "host_s_ms": st.host_s * 1e3, "h2d": st.h2d_bytes, "d2h": st.d2h_bytes,
                          "checksum": st.checksum}))
''' % str(ROOT)
n = sys.argv[1] if len(sys.argv) > 1 else "4096"
genomes = ["001010101001", "100010101001", "101010001001", "000010101001", "001000101001"]
for overlap in ("1", "0"):
    env = dict(os.environ, MMX_OVERLAP=overlap)
    out = subprocess.run([sys.executable, "-c", CHILD, n, *genomes], capture_output=True, text=True, env=env)
    for ln in out.stdout.strip().splitlines():
        row = json.loads(ln)
        row["overlap"] = overlap
        print(json.dumps(row), flush=True)
    if out.returncode != 0:
        print(out.stderr[-500:])
