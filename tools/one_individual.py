"""Three runs of the all-nests-offloaded individual (the bench step) for profiling: python one_individual.py f64|f32 N [matmul_variant]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

dtype = capi.F64 if sys.argv[1] == "f64" else capi.F32
n = int(sys.argv[2])
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
with capi.Context(n=n, dtype=dtype, launch_batching=0, matmul_variant=variant) as ctx:
    for _ in range(3):
        out = ctx.measure("101010101001")
        assert out.status == capi.MEASURED
        print(out.time_s)
