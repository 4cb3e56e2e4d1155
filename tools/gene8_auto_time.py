"""Gene 8 in FP64 auto mode on the application's operands: the form the device picked, time per launch (slice passes and the
guarded FP64-pipe launch included), and the whole individual.  usage: python tools/gene8_auto_time.py [N ...]"""
import sys
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi

sizes = [int(x) for x in sys.argv[1:]] or [4096, 8192]
for n in sizes:
    with capi.Context(n=n, dtype=capi.F64) as ctx:
        out = ctx.measure("101010101001")
        ctx.time_loop(8, 2, True)
        ms = ctx.time_loop(8, 5, True)
        form = ctx.gene8_form()
        best = min(ctx.measure("101010101001").time_s for _ in range(5))
        print(f"N={n} form={form} gene8 {ms:.4f} ms = {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s; individual {best * 1e3:.4f} ms = "
              f"{2 * n ** 3 / best / 1e12:.1f} TFLOP/s", flush=True)
