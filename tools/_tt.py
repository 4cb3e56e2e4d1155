import sys
sys.path.insert(0, "/root/repo")
from paper_1806_01430_b200 import capi
for n in (4096, 8192):
    for dtype in (0, 1):
        with capi.Context(n=n, dtype=dtype, timeout_s=600.0, launch_batching=0) as ctx:
            for _ in range(4):
                ctx.measure("101010101001")
