"""GPU probe of the FP32 tensor-core contraction (variant 30, matmul_tc.cu): error against the float64-exact
product relative to the 1e-6 norm-wise bar, next to the FFMA kernel, and kernel time."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402


def ratio(got, a, bt, c0):
    exact = c0.astype(np.float64) + a.astype(np.float64) @ bt.astype(np.float64).T
    bound = 1e-6 * (np.abs(c0).astype(np.float64) + np.abs(a).astype(np.float64) @ np.abs(bt).astype(np.float64).T)
    err = np.abs(got.astype(np.float64) - exact)
    return float((err / np.maximum(bound, 1e-300)).max()), float(np.sqrt((err ** 2).mean()) / np.sqrt((bound ** 2).mean()))


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [1024, 1000, 2048, 4096]
    for n in sizes:
        rs = np.random.RandomState(n)
        cases = {"random": (rs.uniform(-1, 1, (n, n)).astype(np.float32), rs.uniform(-1, 1, (n, n)).astype(np.float32),
                            rs.uniform(-1, 1, (n, n)).astype(np.float32))}
        i = np.arange(n, dtype=np.float64)
        a = ((i[:, None] + i[None, :]) / n).astype(np.float32)
        b = ((i[:, None] - i[None, :]) / n).astype(np.float32)
        cases["app"] = (a, np.ascontiguousarray(b.T), np.zeros((n, n), np.float32))
        for variant in (30,):
            with capi.Context(n=n, dtype=capi.F32, matmul_variant=variant) as ctx:
                for name, (a_, bt_, c0) in cases.items():
                    ctx.upload(capi.ARRAY_A, a_)
                    ctx.upload(capi.ARRAY_BT, bt_)
                    ctx.upload(capi.ARRAY_C, c0)
                    ctx.run_loop(8)
                    got = ctx.fetch(capi.ARRAY_C)
                    mx, rms = ratio(got, a_, bt_, c0)
                    print(json.dumps({"n": n, "variant": variant, "case": name, "max_err_over_bar": mx, "rms_err_over_bar": rms}), flush=True)
                ms = ctx.time_loop(8, 5, True)
                print(json.dumps({"n": n, "variant": variant, "ms": ms, "TFLOPs": 2.0 * n ** 3 / ms / 1e9}), flush=True)
                if os.environ.get("TC_SCALING") and variant == 30:
                    import time
                    for rows in (128, 512, 1152, 2304, n):   # CTA rows of 128: how does time scale with the number of CTAs?
                        rows = min(rows, n)
                        ctx.run_loop_rows(8, 0, rows)
                        t0 = time.perf_counter()
                        for _ in range(5):
                            ctx.run_loop_rows(8, 0, rows)
                        dt = (time.perf_counter() - t0) / 5
                        print(json.dumps({"n": n, "rows": rows, "ms": dt * 1e3, "TFLOPs": 2.0 * rows * n * n / dt / 1e12}), flush=True)


if __name__ == "__main__":
    main()
