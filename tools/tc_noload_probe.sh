for nl in 0 1; do for m in 14802 14816; do echo "== noload=$nl mode=$m"; MMX_TC_NOLOAD=$nl MMX_TC_MODE=$m python - <<'PY'
import sys, json
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi
for n in (4096, 8192):
    with capi.Context(n=n, dtype=capi.F32, matmul_variant=30) as ctx:
        ctx.measure("101010101001")
        ctx.time_loop(8, 2, True)
        ms = ctx.time_loop(8, 5, True)
        print(json.dumps({"n": n, "ms": round(ms, 4), "TFLOPs": round(2 * n ** 3 / ms / 1e9, 1)}))
PY
done; done
