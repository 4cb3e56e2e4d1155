#!/bin/bash
# Everything the round's numbers come from, in one GPU call: bash tools/round_evidence.sh <tag>   (run under gpurun from the repo root)
tag=${1:-r2}
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > $out/${tag}_gputests.log
timeout 600 python bench.py --impl reference > $out/${tag}_bench_reference.json 2> $out/${tag}_bench_reference.err
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 300 python tools/peaks.py --out $out/${tag}_peaks.json > /dev/null 2>&1
bash tools/profile_round.sh $tag > $out/${tag}_profile_round.log 2>&1
timeout 300 python tools/kernel_times.py --n 4096 --out $out/${tag}_kernel_times_4096.json > $out/${tag}_kt.log 2>&1
timeout 300 python tools/gene8_auto_time.py 4096 8192 16384 32768 > $out/${tag}_gene8.jsonl 2> $out/${tag}_gene8.err
timeout 900 python tools/config5_large_n.py --n 4096 8192 16384 --world 1 2 4 > $out/${tag}_config5.jsonl 2> $out/${tag}_config5.err
timeout 600 python tools/config5_large_n.py --n 32768 --world 1 > $out/${tag}_config5_32768.jsonl 2>> $out/${tag}_config5.err
timeout 600 python tools/config3_residency.py 8192 8.0 8 > $out/${tag}_config3.jsonl 2> $out/${tag}_config3.err
# bench.py under the driver's multi-GPU launch line; with one GPU both ranks share it (gloo, MMX_BENCH_SHARE_DEVICE=1): the code path
# of the 8-GPU run, not a scaling number
gpus=$(nvidia-smi -L | wc -l)
if [ "$gpus" -ge 2 ]; then share=0; else share=1; fi
MMX_BENCH_SHARE_DEVICE=$share timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu-baseline --no-fp32 --no-fp64-pipe --no-fp64-random --no-sustained \
    > $out/${tag}_bench_2ranks.json 2> $out/${tag}_bench_2ranks.err
bash tools/sanitize.sh $tag > /dev/null 2>&1
cat $out/${tag}_gputests.log
