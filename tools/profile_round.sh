#!/bin/bash
# GPU-side evidence for one round: launch list of the bench command, one `ncu --set full` capture of each dominant kernel, boiled
# down ON THE BOX to the per-launch summaries the roofline discussion uses (tools/ncu_summary.py) -- gpurun_out/ is capped at 64 MiB,
# so the .ncu-rep files stay in /tmp except the contraction's, which is small enough to travel.
# Run under gpurun from the repo root:  bash tools/profile_round.sh <tag>
tag=${1:-r2}
out=gpurun_out
rep=/tmp/mmx_ncu_$tag
mkdir -p $out $rep
# every launch of a short bench run with its device time (serialised, cold cache: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sustained --no-fp64-random > $out/${tag}_ncu_bench.log 2>&1
capture() {   # capture <name> <kernel regex> <skip> <count> <command...>
  local name=$1 regex=$2 skip=$3 count=$4; shift 4
  ncu --set full --clock-control none --import-source on -k regex:"$regex" -s $skip -c $count -f -o $rep/${tag}_$name "$@" > $out/${tag}_ncu_$name.log 2>&1
  python tools/ncu_summary.py $rep/${tag}_$name.ncu-rep > $out/${tag}_ncu_${name}_summary.csv 2>> $out/${tag}_ncu_$name.log
}
# the kernels of one FP64 individual at N = 4096 (launch_batching off: plain stream launches): the fused producers (init-a and the
# transpose, which also write the digit planes), the HBM-bound fills, the INT8 contraction as CTA pairs, the guarded FP64-pipe launch, the trace
capture f64 'fill_a_planes|fill2d|b_colexp|transpose_tile|ozaki_auto|matmul_dmma|trace' 9 9 python tools/one_individual.py f64 4096
python tools/ncu_summary.py --traffic $rep/${tag}_f64.ncu-rep 4096 $out/${tag}_ncu_traffic.json >> $out/${tag}_ncu_f64.log 2>&1
# the FP64-pipe contraction itself (variant 4), the FP32 individual, the FP32 split-TF32 path (variant 30)
capture dmma 'matmul_dmma' 2 1 python tools/one_individual.py f64 4096 4
python tools/ncu_summary.py --traffic $rep/${tag}_dmma.ncu-rep 4096 $out/${tag}_ncu_traffic.json >> $out/${tag}_ncu_dmma.log 2>&1
capture f32 'fill_a_planes|transpose_tile|ozaki_auto' 3 3 python tools/one_individual.py f32 4096
capture f32_tf32 'matmul_3xtf32|split_tf32|split_planes' 6 3 python tools/one_individual.py f32 4096 30
python tools/ncu_summary.py --traffic $rep/${tag}_f32_tf32.ncu-rep 4096 $out/${tag}_ncu_traffic.json >> $out/${tag}_ncu_f32_tf32.log 2>&1
# the contraction at the sizes of the other forms (3 x 2 at 8192, 3 x 3 at 16384)
capture ozaki_8192 'ozaki_auto' 1 1 python tools/ozaki_one.py 8192 0
capture ozaki_16384 'ozaki_auto' 1 1 python tools/ozaki_one.py 16384 0
# one report small enough to travel: the contraction at N = 4096 alone
ncu --set full --clock-control none --import-source on -k regex:'ozaki_auto' -s 1 -c 1 -f -o $out/${tag}_prof_ozaki_4096 python tools/ozaki_one.py 4096 0 > /dev/null 2>&1
ls -la $rep $out | tail -30
du -sh $out
