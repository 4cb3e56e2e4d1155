#!/bin/bash
# Everything the round's numbers come from, in one GPU call: bash tools/round_evidence.sh <tag>   (run under gpurun from the repo root)
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > $out/${tag}_gputests.log
timeout 600 python bench.py --impl reference > $out/${tag}_bench_reference.json 2> $out/${tag}_bench_reference.err
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
bash tools/profile_round.sh $tag > $out/${tag}_profile_round.log 2>&1
timeout 300 python tools/kernel_times.py --n 4096 --out $out/${tag}_kernel_times_4096.json > $out/${tag}_kt.log 2>&1
timeout 900 python tools/config5_large_n.py --n 4096 8192 16384 --world 1 2 4 > $out/${tag}_config5.jsonl 2> $out/${tag}_config5.err
timeout 600 python tools/config5_large_n.py --n 32768 --world 1 > $out/${tag}_config5_32768.jsonl 2>> $out/${tag}_config5.err
timeout 600 python tools/config3_residency.py 8192 8.0 8 > $out/${tag}_config3.jsonl 2> $out/${tag}_config3.err
timeout 900 python tools/config4_ga.py 4096 64 40 6.0 16 > $out/${tag}_ga_n4096_64x40.txt 2> $out/${tag}_ga.err
cat $out/${tag}_gputests.log
