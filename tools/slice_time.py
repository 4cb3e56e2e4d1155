"""Per-kernel device times of one FP64 individual at N (ncu launch list is the reference; this is the quick look)."""
import sys
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
with capi.Context(n=n, dtype=capi.F64) as ctx:
    ctx.measure("101010101001")
    for g in (0, 6, 8, 11):
        ctx.time_loop(g, 2, True)
        print("gene", g, round(ctx.time_loop(g, 10, True) * 1e3, 1), "us")
    print("individual", min(ctx.measure("101010101001").time_s for _ in range(5)) * 1e6, "us", "form", ctx.gene8_form())
