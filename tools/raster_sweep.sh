#!/bin/bash
# Tile-order sweep of the gene-8 kernels: kernel time (CUDA events, no profiler) and DRAM traffic (ncu) per
# MMX_RASTER_GROUP value.  Run under gpurun from the repo root:  bash tools/raster_sweep.sh <tag> [N ...]
tag=${1:-raster}; shift
sizes=${@:-4096}
out=gpurun_out/${tag}_raster.txt
: > $out
for n in $sizes; do
  for g in 1 4 8 16 32 0; do
    echo "== N=$n group=$g (0 = auto)" >> $out
    MMX_RASTER_GROUP=$g python - $n >> $out 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi
n = int(sys.argv[1])
for dtype, name in ((capi.F64, "f64"), (capi.F32, "f32")):
    with capi.Context(n=n, dtype=dtype) as ctx:
        assert ctx.measure("101010101001").status == capi.MEASURED
        ctx.time_loop(8, 2, True)
        ms = ctx.time_loop(8, 5, True)
        print(json.dumps({"n": n, "dtype": name, "ms": round(ms, 4), "TFLOPs": round(2 * n ** 3 / ms / 1e9, 2)}))
PY
    for dt in f64 f32; do
      MMX_RASTER_GROUP=$g ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:'matmul_dmma|matmul_3xtf32' -s 1 -c 1 --csv python tools/one_individual.py $dt $n 2>/dev/null \
        | grep -E 'dram__bytes|gpu__time' | awk -F'","' -v dt=$dt '{print dt, $5, $(NF-2), $(NF-1), $NF}' >> $out
    done
  done
done
cat $out
