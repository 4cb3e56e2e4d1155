#!/usr/bin/env python
"""A/B timing of the gene-8 kernel variants (CUDA events, L2 flushed)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[4096])
ap.add_argument("--iters", type=int, default=5)
args = ap.parse_args()
for n in args.n:
    for dtype, name, variants in ((capi.F64, "f64", (1, 0, 20, 2, 6, 8)), (capi.F32, "f32", (1, 0, 22))):
        for numerics in (capi.FAST, capi.STRICT):
            for v in variants:
                if numerics == capi.STRICT and v not in (0, 1, 20):
                    continue
                with capi.Context(n=n, dtype=dtype, numerics=numerics, matmul_variant=v) as ctx:
                    assert ctx.measure("101010101001").status == capi.MEASURED
                    ctx.time_loop(8, 2, True)
                    ms = ctx.time_loop(8, args.iters, True)
                    print(json.dumps({"n": n, "dtype": name, "numerics": "strict" if numerics else "fast", "variant": v,
                                      "ms": round(ms, 4), "TFLOPs": round(2 * n ** 3 / ms / 1e9, 2)}), flush=True)
