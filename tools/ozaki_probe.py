"""GPU probe of the FP64 tensor-core contraction (variants 40 / 41, matmul_ozaki.cu): bit-exactness on the application's
inputs, error against the 1e-12 norm-wise bar on random inputs next to the DMMA kernel, and kernel time.
python tools/ozaki_probe.py [N ...]"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import cpu  # noqa: E402
from paper_1806_01430_b200 import capi  # noqa: E402


def ratio(got, a, bt, c0):
    exact = c0.astype(np.longdouble) + a.astype(np.longdouble) @ bt.astype(np.longdouble).T if a.shape[0] <= 512 else c0 + a @ bt.T
    bound = 1e-12 * (np.abs(c0) + np.abs(a) @ np.abs(bt).T)
    err = np.abs(got.astype(np.longdouble) - exact).astype(np.float64)
    return float((err / np.maximum(bound, 1e-300)).max())


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [256, 300, 1024, 4096]
    for n in sizes:
        rs = np.random.RandomState(n)
        a, bt, c0 = rs.uniform(-1, 1, (n, n)), rs.uniform(-1, 1, (n, n)), rs.uniform(-1, 1, (n, n))
        # rows with very different magnitudes: the per-row exponents must absorb them
        a *= np.exp2(rs.randint(-20, 20, (n, 1)).astype(np.float64))
        bt *= np.exp2(rs.randint(-20, 20, (n, 1)).astype(np.float64))
        for variant in (4, 40, 41):
            with capi.Context(n=n, dtype=capi.F64, matmul_variant=variant, timeout_s=120.0) as ctx:
                out = ctx.measure("101010101001")
                assert out.status == capi.MEASURED, capi.STATUS_NAMES[out.status]
                got = ctx.fetch(capi.ARRAY_C)
                exact_app = all(np.array_equal(got[r0:r0 + 256].view(np.uint64), cpu.closed_form_c(n, r0, min(n, r0 + 256)).view(np.uint64))
                                for r0 in range(0, n, 256)) if n & (n - 1) == 0 else None
                ctx.upload(capi.ARRAY_A, a)
                ctx.upload(capi.ARRAY_BT, bt)
                ctx.upload(capi.ARRAY_C, c0)
                ctx.run_loop(8)
                r = ratio(ctx.fetch(capi.ARRAY_C), a, bt, c0)
                ctx.time_loop(8, 2, True)
                ms = ctx.time_loop(8, 5, True)
                print(json.dumps({"n": n, "variant": variant, "app_inputs_bit_exact": exact_app, "individual_us": out.time_s * 1e6,
                                  "random_max_err_over_1e-12_bar": r, "ms": ms, "TFLOPs": 2.0 * n ** 3 / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
