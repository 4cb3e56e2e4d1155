#!/usr/bin/env python
"""time of a genome with a CPU-mapped matmul nest, alone and with every other slot busy, pinned (default) and not.
python tools/pinning_probe.py [N] [slots]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 8
genome = "101010100001"
for pin in (1, 0):
    with capi.Context(n=n, num_slots=slots, devices=[0] * slots, host_threads=1, timeout_s=60.0, pin_host=pin) as ctx:
        alone = sorted(ctx.measure(genome, slot=0).time_s for _ in range(5))
        crowded = []
        for _ in range(5):
            outs = ctx.measure_batch([genome] * slots)
            crowded.append(sorted(o.time_s for o in outs))
        worst = sorted(c[-1] for c in crowded)
        best = sorted(c[0] for c in crowded)
        st = [ctx.stats(s) for s in range(slots)]
        print(json.dumps({"n": n, "slots": slots, "pin_host": pin, "cpus": os.cpu_count(), "alone_ms": alone[2] * 1e3,
                          "crowded_worst_slot_ms": worst[2] * 1e3, "crowded_best_slot_ms": best[2] * 1e3,
                          "ratio_worst": worst[2] / alone[2], "slot_first_cpus": [s.host_first_cpu for s in st],
                          "slot_cpus": [s.host_cpus for s in st], "loadavg": st[0].host_loadavg}), flush=True)
