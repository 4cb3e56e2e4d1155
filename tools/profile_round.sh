#!/bin/bash
# GPU-side evidence for one round: launch list of the bench command, one `ncu --set full` capture of each dominant
# kernel, clocks.  Run under gpurun from the repo root:  bash tools/profile_round.sh <tag>
tag=${1:-r2}
out=gpurun_out
mkdir -p $out
# every launch of a short bench run with its device time (serialised, cold cache: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sustained --no-fp64-random > $out/${tag}_ncu_bench.log 2>&1
# the kernels of one FP64 individual at N = 4096 (launch_batching off: plain stream launches): the fused producers (init-a and the
# transpose, which also write the digit planes), the HBM-bound fills, the INT8 contraction as CTA pairs, the trace
ncu --set full --clock-control none --import-source on -k regex:'fill_a_planes|fill2d|transpose_tile|ozaki_auto|matmul_dmma|trace' -s 9 -c 9 -f \
    -o $out/${tag}_prof_f64 python tools/one_individual.py f64 4096 > $out/${tag}_ncu_f64.log 2>&1
# the FP64-pipe contraction itself (variant 4) and the FP32 split-TF32 path (variant 30)
ncu --set full --clock-control none --import-source on -k regex:'matmul_dmma' -s 2 -c 1 -f \
    -o $out/${tag}_prof_dmma python tools/one_individual.py f64 4096 4 > $out/${tag}_ncu_dmma.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'matmul_3xtf32|split_tf32|split_planes' -s 6 -c 3 -f \
    -o $out/${tag}_prof_f32 python tools/one_individual.py f32 4096 30 > $out/${tag}_ncu_f32.log 2>&1
# the contraction at the sizes of the other forms (3 x 2 at 8192, 3 x 3 at 16384)
ncu --set full --clock-control none --import-source on -k regex:'ozaki_auto' -s 1 -c 1 -f \
    -o $out/${tag}_prof_ozaki_8192 python tools/ozaki_one.py 8192 0 > $out/${tag}_ncu_ozaki_8192.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'ozaki_auto' -s 1 -c 1 -f \
    -o $out/${tag}_prof_ozaki_16384 python tools/ozaki_one.py 16384 0 > $out/${tag}_ncu_ozaki_16384.log 2>&1
ls -la $out | tail -12
