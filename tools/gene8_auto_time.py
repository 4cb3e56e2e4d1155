import sys
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi
for n in (4096, 8192):
    with capi.Context(n=n, dtype=capi.F64) as ctx:
        out = ctx.measure("101010101001"); ctx.time_loop(8, 2, True)
        ms = ctx.time_loop(8, 5, True)
        out = ctx.measure("101010101001")
        print(n, "gene8 ms", round(ms, 4), "TFLOP/s", round(2 * n ** 3 / ms / 1e9, 1), "individual ms", round(out.time_s * 1e3, 4))
