#!/bin/bash
# GPU-side evidence for one round: launch list of the bench command, one `ncu --set full` capture of each dominant
# kernel, clocks.  Run under gpurun from the repo root:  bash tools/profile_round.sh <tag>
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
# every launch of a short bench run with its device time (serialised, cold cache: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/${tag}_ncu_bench.log 2>&1
# the FP64 contraction (DMMA), the FP32 contraction (tcgen05) and the HBM-bound kernels of one individual
ncu --set full --clock-control none --import-source on -k regex:'matmul_dmma|transpose_tile|fill2d|trace' -s 12 -c 6 -f \
    -o $out/${tag}_prof_f64 python tools/one_individual.py f64 4096 > $out/${tag}_ncu_f64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'matmul_3xtf32|split_tf32|split_planes' -s 6 -c 3 -f \
    -o $out/${tag}_prof_f32 python tools/one_individual.py f32 4096 30 > $out/${tag}_ncu_f32.log 2>&1   # variant 30: the split-TF32 path itself
ls -la $out | tail -8
ncu --set full --clock-control none --import-source on -k regex:'ozaki' -s 3 -c 3 -f \
    -o $out/${tag}_prof_ozaki python tools/ozaki_one.py 4096 0 > $out/${tag}_ncu_ozaki.log 2>&1
