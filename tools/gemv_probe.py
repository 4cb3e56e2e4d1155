"""GEMV (gene 9) timing, L2 flushed between launches: python tools/gemv_probe.py [N ...]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [4096]:
    for dtype, e, name in ((capi.F64, 8, "f64"), (capi.F32, 4, "f32")):
        with capi.Context(n=n, dtype=dtype) as ctx:
            assert ctx.measure("101010101001").status == capi.MEASURED
            ctx.time_loop(9, 3, True)
            ms = ctx.time_loop(9, 20, True)
            warm = ctx.time_loop(9, 20, False)
            print(json.dumps({"n": n, "dtype": name, "ms_flushed": ms, "GBps_flushed": e * n * n / ms / 1e6, "ms_warm_l2": warm,
                              "GBps_warm_l2": e * n * n / warm / 1e6}), flush=True)
