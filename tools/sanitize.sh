#!/bin/bash
# compute-sanitizer passes over small individuals (memcheck: out-of-bounds / misaligned accesses; racecheck: shared-memory
# hazards; synccheck: barrier misuse).  Run under gpurun from the repo root:  bash tools/sanitize.sh <tag>
tag=${1:-r2}
out=gpurun_out/${tag}_sanitizer.txt
: > $out
for tool in memcheck synccheck; do
  for cfg in "f64 1024" "f32 1024" "f32 1024 30" "f64 2048" "f64 256"; do   # 1024+: INT8 forms (persistent tcgen05 kernel, TMA reductions); "30": split TF32
    echo "== compute-sanitizer --tool $tool  one_individual.py $cfg" >> $out
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 python tools/one_individual.py $cfg 2>&1 | grep -E "ERROR SUMMARY|Error|error|Invalid|hazard|=========.*at " | head -12 >> $out
  done
done
for tool in memcheck synccheck; do   # every pair form (cta_group::2 bodies, 128- and 96-wide tiles) and two one-CTA forms on synthetic operands
  echo "== compute-sanitizer --tool $tool  ozaki_forms_once.py" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python tools/ozaki_forms_once.py 2>&1 | grep -E "ERROR SUMMARY|Error|error|Invalid|hazard|=========.*at |digits" | head -20 >> $out
done
echo "== compute-sanitizer --tool racecheck  one_individual.py f64 256 (FP64 pipe kernels, fills, transpose, trace)" >> $out
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python tools/one_individual.py f64 256 2>&1 | grep -E "RACECHECK SUMMARY|hazard|Error" | head -12 >> $out
cat $out
