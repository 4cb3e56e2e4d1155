#!/usr/bin/env python
"""Per-loop kernel timings (CUDA events, L2 flushed between launches) against their rooflines."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402


def algorithmic(gene: int, n: int, e: int):
    """(bytes, flops) one launch of loop `gene` must move / compute."""
    if gene in (0, 2, 4):
        return e * n * n, 0
    if gene in (1, 3, 5):
        return e * n, 0
    if gene == 6:
        return 2 * e * n * n, 0
    if gene == 7:
        return 2 * e * n, 0
    if gene == 8:
        return 4 * e * n * n, 2 * n ** 3
    if gene == 9:
        return e * n * n + 3 * e * n, 2 * n * n
    if gene == 10:
        return 2 * e * n + 2 * e, 2 * n
    return e * n, n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[4096])
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out")
    args = ap.parse_args()
    rows = []
    for n in args.n:
        for dtype, e in ((capi.F64, 8), (capi.F32, 4)):
            for numerics in (capi.FAST, capi.STRICT):
                variants = (0, 1, 2) if (dtype == capi.F64 and numerics == capi.FAST) else ((0, 1) if numerics == capi.FAST else (1,))
                for variant in variants:
                    with capi.Context(n=n, dtype=dtype, numerics=numerics, matmul_variant=variant) as ctx:
                        assert ctx.measure("101010101001").status == capi.MEASURED  # populate arrays, warm up
                        for gene in range(12):
                            if numerics == capi.STRICT and gene not in (8, 9, 10, 11):
                                continue
                            if variant != 1 and gene != 8:
                                continue
                            ctx.time_loop(gene, 2, True)
                            ms = ctx.time_loop(gene, args.iters if gene != 8 else max(3, args.iters // 3), True)
                            by, fl = algorithmic(gene, n, e)
                            rows.append({"n": n, "dtype": "f64" if dtype == capi.F64 else "f32",
                                         "numerics": "strict" if numerics else "fast", "variant": variant, "gene": gene,
                                         "ms": ms, "GBps": by / ms / 1e6, "TFLOPs": fl / ms / 1e9})
                            print(json.dumps(rows[-1]), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
