"""FP32 gene 8 at N=4096: auto mode (INT8 forms, split TF32 as the guarded fallback) against matmul_variant 30 (split TF32 always).
MMX_F32_INT8=0 switches the INT8 forms off.  usage: python tools/f32_probe.py"""
import sys, os
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi
n = 4096
for variant in (0, 30):
    with capi.Context(n=n, dtype=capi.F32, matmul_variant=variant) as ctx:
        ctx.measure("101010101001"); ctx.time_loop(8, 2, True)
        ms = ctx.time_loop(8, 5, True)
        best = min(ctx.measure("101010101001").time_s for _ in range(5))
        print("variant", variant, "form", ctx.gene8_form(), "gene8 ms", round(ms, 4), round(2*n**3/ms/1e9, 1), "individual ms", round(best*1e3, 4), round(2*n**3/best/1e12, 1), flush=True)
