#!/bin/bash
# Where the pair body's tile boundary goes: MMX_OZ_TRACE=1 makes the leader CTA of pair 0 record its SM clock at the hand-over points of
# every tile (matmul_ozaki.cu, OzPArgs::trace); run under gpurun from the repo root: bash tools/handover_trace.sh <tag>
tag=${1:-r2f}
out=gpurun_out
mkdir -p $out
for dbg in 0 4096 1 2049; do
  echo "MMX_OZ_DEBUG=$dbg" >> $out/${tag}_handover.txt
  MMX_OZ_TRACE=1 MMX_OZ_DEBUG=$dbg timeout 300 python tools/gene8_auto_time.py 4096 2>&1 | grep -E "oztrace|contraction_ms" | tail -9 >> $out/${tag}_handover.txt
done
for dbg in 0 4096; do
  echo "MMX_OZ_DEBUG=$dbg (no trace)" >> $out/${tag}_handover.txt
  MMX_OZ_DEBUG=$dbg timeout 300 python tools/gene8_auto_time.py 4096 8192 2>&1 | tail -2 >> $out/${tag}_handover.txt
done
cat $out/${tag}_handover.txt
