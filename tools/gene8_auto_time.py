"""Gene 8 in FP64 auto mode on the application's operands: the form the device picked, time per launch of the whole nest (slice
passes and the guarded FP64-pipe launch included), the contraction kernel alone against the measured INT8 issue peak, and the
whole individual.  usage: python tools/gene8_auto_time.py [N ...]"""
import json
import sys
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi

sizes = [int(x) for x in sys.argv[1:]] or [4096, 8192]
peak = capi.peak_probe(capi.PEAK_UMMA_I8)
for n in sizes:
    with capi.Context(n=n, dtype=capi.F64, timeout_s=600.0) as ctx:
        out = ctx.measure("101010101001")
        ctx.time_loop(8, 2, True)
        ms = ctx.time_loop(8, 3 if n > 8192 else 5, True)
        form = ctx.gene8_form()
        sa, sb, lv = form // 100, form // 10 % 10, form % 10
        products = sum(1 for t in range(1, sa + 1) for u in range(1, sb + 1) if t + u <= lv + 1)
        msk = ctx.time_gene8_contraction(3 if n > 8192 else 5, True)
        best = min(ctx.measure("101010101001").time_s for _ in range(5))
        tops = products * 2 * n ** 3 / msk / 1e9
        print(json.dumps({"n": n, "form": form, "nest_ms": ms, "nest_tflops": 2 * n ** 3 / ms / 1e9, "contraction_ms": msk,
                          "contraction_tops": tops, "int8_issue_peak_tops": peak, "frac": tops / peak,
                          "individual_ms": best * 1e3, "app_tflops": 2 * n ** 3 / best / 1e12}), flush=True)
