#!/usr/bin/env python
"""BASELINE config 3: the matrix application at N=8192 FP64 under mixed GPU/CPU genomes -- what the device-residency
planner moves (bytes up / down per run against its independently derived lower bound), and what the individual costs.
Genomes are SURVEY 8d's list: every array hand-off of the program appears at least once."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

GENOMES = [
    ("101010101001", "all six nests on the GPU"),
    ("001010101001", "init-a on the CPU: a goes up"),
    ("100010101001", "init-b on the CPU: b goes up"),
    ("101000101001", "zero-c on the CPU: c goes up"),
    ("101010001001", "transpose on the CPU: b down, bt up"),
    ("101010101000", "trace on the CPU: only the diagonal of c comes down"),
    ("000000001001", "only matmul + trace on the GPU: a, bt, c go up"),
    ("000000001000", "only matmul on the GPU: a, bt, c up, diagonal down"),
    ("101010100001", "matmul on the CPU: a, bt, c down, diagonal up (hits the timeout budget)"),
    ("010000000000", "init-a inner loop only: N row-fill launches, a comes down for the CPU matmul (timeout)"),
    ("101010100101", "matmul as N GEMV launches (gene 9)"),
    ("101010010001", "transpose as N row launches (gene 7) and matmul on the CPU (timeout)"),
    ("101001101001", "zero-c as N row launches (gene 5)"),
]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    timeout_s = float(sys.argv[2]) if len(sys.argv) > 2 else 8.0
    host_threads = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    rows = []
    with capi.Context(n=n, dtype=capi.F64, timeout_s=timeout_s, host_threads=host_threads) as ctx:
        ctx.measure("101010101001")   # warm-up: module load, pinned allocations happen on first need per genome
        for genome, what in GENOMES:
            plan = capi.plan(genome, n, capi.F64)
            out = ctx.measure(genome)
            st = ctx.stats()
            row = {"n": n, "genome": genome, "what": what, "status": capi.STATUS_NAMES[out.status], "time_s": out.time_s,
                   "h2d_bytes": int(st.h2d_bytes), "d2h_bytes": int(st.d2h_bytes),
                   "h2d_lower_bound": int(plan.h2d_lower_bound), "d2h_lower_bound": int(plan.d2h_lower_bound),
                   "meets_lower_bound": int(plan.h2d_bytes) == int(plan.h2d_lower_bound) and int(plan.d2h_bytes) == int(plan.d2h_lower_bound),
                   "kernel_launches": int(st.kernel_launches), "graph_launches": int(st.graph_launches),
                   "gpu_ms": st.gpu_ms, "host_s": st.host_s, "app_gflops": 2.0 * n ** 3 / out.time_s / 1e9 if out.status == 0 else None}
            rows.append(row)
            print(json.dumps(row), flush=True)
    print(json.dumps({"summary": "config3", "n": n, "timeout_s": timeout_s, "host_threads": host_threads,
                      "all_plans_meet_lower_bound": all(r["meets_lower_bound"] for r in rows)}))


if __name__ == "__main__":
    main()
