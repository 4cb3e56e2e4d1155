#!/usr/bin/env python
"""time of a genome with a CPU-mapped matmul nest on slot 0, alone and with every other slot running the all-CPU genome
(host work only: on a one-GPU box the slots share the device, and neighbours with device work would queue in front of the measured
slot's kernels and copies), pinned (default) and not.  python tools/pinning_probe.py [N] [slots]"""
import json
import os
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 8
genome = "101010100001"
for pin in (1, 0):
    with capi.Context(n=n, num_slots=slots, devices=[0] * slots, host_threads=1, timeout_s=60.0, pin_host=pin) as ctx:
        for s in range(slots):
            ctx.measure(genome, slot=s)      # first use of a slot allocates its pinned host mirrors
        alone = sorted(ctx.measure(genome, slot=0).time_s for _ in range(15))
        stop = threading.Event()

        def neighbour(slot):
            while not stop.is_set():
                ctx.measure("000000000000", slot=slot)

        threads = [threading.Thread(target=neighbour, args=(s,)) for s in range(1, slots)]
        for t in threads:
            t.start()
        crowded = sorted(ctx.measure(genome, slot=0).time_s for _ in range(15))
        stop.set()
        for t in threads:
            t.join()
        st = [ctx.stats(s) for s in range(slots)]
        print(json.dumps({"n": n, "slots": slots, "pin_host": pin, "cpus": os.cpu_count(), "alone_median_ms": alone[7] * 1e3,
                          "crowded_median_ms": crowded[7] * 1e3, "crowded_max_ms": crowded[-1] * 1e3, "ratio_median": crowded[7] / alone[7],
                          "ratio_max": crowded[-1] / alone[7], "slot_first_cpus": [s.host_first_cpu for s in st],
                          "slot_cpus": [s.host_cpus for s in st]}), flush=True)
