import sys
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi
n = int(sys.argv[1]); v = int(sys.argv[2])
with capi.Context(n=n, dtype=capi.F64, matmul_variant=v, launch_batching=0) as ctx:
    for _ in range(2):
        out = ctx.measure("101010101001"); print(out.time_s)
