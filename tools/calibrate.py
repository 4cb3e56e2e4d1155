#!/usr/bin/env python
"""Cost-model calibration on a real GPU.

1. measures EVERY feasible genome of the matrix application (648 of 4096) at size N through the C ABI -- the exhaustive
   ground truth for "did the GA find the best pattern";
2. fits the executor's plan model and projects it onto the reference's cost-model file (mmxhost/calibrate.hpp);
3. runs the GA (a) on the real CUDA evaluator and (b) on a SimBackend replaying the calibrated file, and reports where each
   lands relative to the measured optimum.
python tools/calibrate.py [N] [out_prefix] [repetitions]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1806_01430_b200 import capi, hostapi as H  # noqa: E402


def genome_of(mask):
    return "".join("1" if (mask >> k) & 1 else "0" for k in range(12))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    prefix = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/calibration_n{n}"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    feasible = [genome_of(m) for m in range(4096) if capi.plan(genome_of(m), n, capi.F64).feasible]
    assert len(feasible) == 648
    t0 = time.perf_counter()
    measured = {}
    with capi.Context(n=n, dtype=capi.F64, timeout_s=30.0, repetitions=reps, warmup=1) as ctx:
        for g in feasible:
            out = ctx.measure(g)
            if out.status == capi.MEASURED:
                measured[g] = out.time_s
    sweep_s = time.perf_counter() - t0
    genomes = sorted(measured, key=measured.get)
    times = [measured[g] for g in genomes]
    cal = H.calibrate(genomes, times, n)
    Path(prefix + "_model.json").write_text(cal["model_json"])
    plan_t = H.plan_model_times(cal["plan"], n)
    idx = {g: sum(1 << k for k, ch in enumerate(g) if ch == "1") for g in genomes}
    pred = np.array([plan_t[idx[g]] for g in genomes])
    meas = np.array(times)
    rank_of = {g: r for r, g in enumerate(genomes)}
    # Spearman rank correlation between model and measurement over all measured genomes
    pr = np.argsort(np.argsort(pred))
    spearman = float(np.corrcoef(pr, np.arange(len(genomes)))[0, 1])

    api = H.mine()
    ga = {}
    for pop, gens in ((12, 12), (64, 40)):
        t1 = time.perf_counter()
        with H.Evaluator.from_cuda(api, n=n, dtype=capi.F64, timeout_s=30.0, repetitions=reps, warmup=1, devices=(0,)) as ev:
            real = ev.run_ga(population=pop, generations=gens, seed=1)
            counters = ev.counters()
        real_wall = time.perf_counter() - t1
        with H.Evaluator.from_sim(api, prefix + "_model.json") as ev:
            sim = ev.run_ga(population=pop, generations=gens, seed=1)
        rows = real["csv"].splitlines()[1:]
        # first generation whose best time is within 5 % of the exhaustive measured optimum
        hit = next((int(r.split(",")[0]) for r in rows if float(r.split(",")[1]) <= 1.05 * meas[0]), None)
        ga[f"{pop}x{gens}"] = {
            "real_best_genome": real["best_genome"], "real_best_s": real["best_s"], "real_best_rank_in_exhaustive_sweep": rank_of.get(real["best_genome"]),
            "real_best_over_measured_optimum": real["best_s"] / meas[0], "generation_within_5pct_of_optimum": hit,
            "real_wall_s": real_wall, "real_distinct_genomes": counters["distinct"],
            "sim_best_genome": sim["best_genome"], "sim_best_rank_in_exhaustive_sweep": rank_of.get(sim["best_genome"]),
            "sim_best_measured_s": measured.get(sim["best_genome"]),
            "sim_best_measured_over_optimum": (measured.get(sim["best_genome"]) or float("nan")) / meas[0]}
    report = {
        "n": n, "dtype": "f64", "repetitions": reps, "feasible_genomes": len(feasible), "measured": len(genomes), "sweep_wall_s": sweep_s,
        "measured_optimum": {"genome": genomes[0], "time_s": times[0]}, "measured_top5": [[g, measured[g]] for g in genomes[:5]],
        "all_cpu_genome_s": measured.get("0" * 12), "speedup_of_optimum_vs_all_cpu": (measured.get("0" * 12) or float("nan")) / times[0],
        "fit": cal["report"], "plan_model": {"serial_s": cal["plan"][0], "cpu_s": list(cal["plan"][1:7]), "loop_s": list(cal["plan"][7:19]),
                                              "h2d_GBps": 1e-9 / cal["plan"][19] if cal["plan"][19] > 0 else None,
                                              "d2h_GBps": 1e-9 / cal["plan"][20] if cal["plan"][20] > 0 else None,
                                              "per_transfer_s": cal["plan"][21]},
        "plan_model_best": cal["plan_best"], "plan_model_best_rank_in_exhaustive_sweep": rank_of.get(cal["plan_best"]),
        "cost_model_best": cal["cost_best"], "cost_model_best_rank_in_exhaustive_sweep": rank_of.get(cal["cost_best"]),
        "median_abs_rel_err": float(np.median(np.abs(pred - meas) / meas)), "spearman_model_vs_measured": spearman,
        "ga": ga, "model_file": prefix + "_model.json"}
    Path(prefix + ".json").write_text(json.dumps(report, indent=1) + "\n")
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
