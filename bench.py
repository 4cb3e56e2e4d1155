#!/usr/bin/env python
"""bench.py -- the matrix application under the all-nests-offloaded genome, N=4096 FP64 (BASELINE.json
configs[1]), one process per GPU.

A *step* is one individual: one full pass of the application (init a, init b, zero c, transpose,
matmul, trace) under genome 101010101001 through the C ABI (`mmx_measure`, what the reference's
EvalBackend::measure would call).  Metric: matrix-app GFLOP/s = 2 N^3 / time.

  value   device-resident throughput: 2N^3 * steps / sum of the per-step CUDA-event times of the
          whole individual (events recorded on the library's own stream), max over ranks
  e2e     the same steps timed by the host clock around the C-ABI calls, barrier +
          torch.cuda.synchronize() on both sides: includes planning, launches, the D2H of the checksum.
          The program generates its own inputs (matmul.c:8-18), so for this genome the planner moves
          0 bytes up and 8 bytes down per step; `e2e_mixed` adds a genome with host-produced operands.
  roofline  dominant kernel (the FP64 contraction, gene 8: on this workload the INT8 tensor-core form) timed live with CUDA events
  cpu_baseline  the oracle port (oracle/matmul_oracle.c) on this box's host cores, bounded sample

`--impl reference` times the reference's CPU implementation of the same path (the oracle port of
fixtures/matmul.c with runtime N; the fixture itself is hard-wired to N=256) on the host cores.
With N > 1 GPUs every rank runs its own individuals (population sharding, no collective on the
data path); value is the job total; scaling is weak.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GENOME_ALL_NESTS = "101010101001"   # depth-0 loop of each of the six nests
GENOME_MIXED = "001010101001"       # init-a on the CPU => a crosses the bus once per step


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--size", dest="n", type=int, default=4096, help="matrix size (use --size under torchrun: its own parser finds --n ambiguous)")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the FP32 arm of the configuration")
    ap.add_argument("--no-fp64-pipe", action="store_true", help="skip the arm that forces gene 8 onto the FP64 pipe (DMMA)")
    ap.add_argument("--no-fp64-random", action="store_true", help="skip the arm with uniform(-1,1) operands")
    ap.add_argument("--no-sustained", action="store_true", help="skip the >= 3 s sustained block")
    ap.add_argument("--sustained-seconds", type=float, default=3.0)
    ap.add_argument("--ga", action="store_true", help="run the config-4 GA block (64 x 40, seed 1) also on one GPU (on by default with --gpus > 1)")
    ap.add_argument("--no-multi", action="store_true", help="with --gpus > 1: skip the config-4 (GA) and config-5 (row-sharded) blocks")
    ap.add_argument("--multi-budget", type=float, default=420.0,
                    help="seconds the multi-GPU blocks may take before rank 0 prints the line without them and every rank leaves")
    ap.add_argument("--ga-population", type=int, default=64)
    ap.add_argument("--ga-generations", type=int, default=40)
    ap.add_argument("--ga-timeout", type=float, default=2.0, help="budget per individual in the GA block (a run over it scores the budget)")
    ap.add_argument("--ga-wait-timeouts", action="store_true", help="GA block: wait out every hopeless run (mmx_config.early_timeout = 0), as the "
                                                                     "reference's process timeout does")
    ap.add_argument("--rowshard-n", type=int, nargs="*", default=[16384, 32768], help="sizes of the row-sharded block (config 5)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        sm, smax, reasons = [], None, set()
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(n: int, dtype: int, cores: int) -> dict:
    """The oracle port on the host cores: whole application, matmul nest sampled on its first rows."""
    from oracle import cpu
    flops = 2.0 * n ** 3
    per_row_s = 2.0 * n * n / 2.0e9            # ~2 GFLOP/s per core, only to size the sample
    rows = int(min(n, max(cores, (12.0 / per_row_s) * cores)))   # ~12 s of matmul work
    r = cpu.time_app(n, dtype, cores, rows)
    other = sum(v for k, v in r["seconds"].items() if k != "matmul")
    total = other + r["seconds"]["matmul"] * n / r["matmul_rows"]
    out = {"value": flops / total / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "port",
           "sample": f"all six nests at N={n}; matmul nest timed on rows [0,{r['matmul_rows']}) of {n} and scaled "
                     f"(every row costs the same 2N^2 flop); {cores} host threads, gcc -O2 -ffp-contract=off",
           "app_seconds_scaled": total, "nest_seconds": r["seconds"]}
    if cores > 1:   # the faithful single-thread figure (the reference program has no threading)
        rows1 = int(min(n, max(1, 4.0 / per_row_s)))
        r1 = cpu.time_app(n, dtype, 1, rows1)
        t1 = sum(v for k, v in r1["seconds"].items() if k != "matmul") + r1["seconds"]["matmul"] * n / r1["matmul_rows"]
        out["single_thread_value"] = flops / t1 / 1e9
        out["single_thread_app_seconds_scaled"] = t1
    return out


def run_reference(args):
    rank, _, _ = dist_env()
    if rank != 0:
        return
    from paper_1806_01430_b200 import build
    build.build_oracle()
    n, dtype = args.n, 0 if args.dtype == "f64" else 1
    cores = os.cpu_count() or 1
    from oracle import cpu
    flops = 2.0 * n ** 3
    # calibrate the cost of one matmul row on this box, then size each step's sample so that the whole
    # --steps/--warmup run stays within ~150 s (at most ~4 s of matmul per step)
    cal_rows = min(n, 4 * cores)
    cal = cpu.time_app(n, dtype, cores, cal_rows)
    per_row_wall = max(cal["seconds"]["matmul"] / cal_rows, 1e-9)      # wall seconds per row with all threads busy
    step_budget_s = min(4.0, 150.0 / max(1, args.steps + args.warmup))
    rows = int(min(n, max(cores, step_budget_s / per_row_wall)))
    times = []
    for it in range(args.warmup + args.steps):
        r = cpu.time_app(n, dtype, cores, rows)
        t = sum(v for k, v in r["seconds"].items() if k != "matmul") + r["seconds"]["matmul"] * n / r["matmul_rows"]
        if it >= args.warmup:
            times.append(t)
    ms = 1e3 * sum(times) / len(times)
    value = flops / (ms * 1e-3) / 1e9
    # the reference program itself has no threading (fixtures/matmul.c): the same nests on ONE core, matmul on ~4 s worth of rows
    rows1 = int(min(n, max(1, 4.0 / (per_row_wall * cores))))
    r1 = cpu.time_app(n, dtype, 1, rows1)
    t1 = sum(v for k, v in r1["seconds"].items() if k != "matmul") + r1["seconds"]["matmul"] * n / r1["matmul_rows"]
    sample = (f"per step: all six nests at N={n}, matmul nest on rows [0,{rows}) of {n} scaled to the full nest; "
              f"{cores} host threads; oracle port of fixtures/matmul.c (the fixture is fixed at N=256)")
    line = {
        "impl": "reference", "metric": "matrix_app_gflops", "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (the program generates its own inputs)",
        "config": {"workload": f"matrix app N={n} {args.dtype}, all six nests (reference CPU path)", "n": n},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "port", "sample": sample,
                         "single_thread_value": flops / t1 / 1e9, "single_thread_app_seconds_scaled": t1,
                         "single_thread_sample": f"all six nests on one core, matmul nest on rows [0,{rows1}) of {n} scaled: the reference "
                                                 "program as written (fixtures/matmul.c has no threading)"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def load_measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except ValueError:
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1806_01430_b200 import capi

    rank, local_rank, world = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the product has no CPU fallback")
    # MMX_BENCH_SHARE_DEVICE=1 is a test hook for one-GPU boxes: every rank uses cuda:0 and the process group is gloo (NCCL refuses
    # two ranks on one device); everything else -- the sharding, the IPC handles, the barriers -- is the code the 8-GPU run uses
    share = os.environ.get("MMX_BENCH_SHARE_DEVICE") == "1"
    device = 0 if share else local_rank
    torch.cuda.set_device(device)
    ctl = None            # gloo group for host-side control (handles, barriers, outcomes): the data path never uses a collective
    red_dev = "cuda"
    if world > 1:
        if share:
            dist.init_process_group("gloo")
            ctl, red_dev = dist.group.WORLD, "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
            ctl = dist.new_group(backend="gloo")
    local_rank = device

    n, dtype = args.n, capi.F64 if args.dtype == "f64" else capi.F32
    esz = 8 if dtype == capi.F64 else 4
    flops = 2.0 * n ** 3

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = capi.Context(n=n, dtype=dtype, devices=[local_rank], timeout_s=600.0)
    plan = capi.plan(GENOME_ALL_NESTS, n, dtype)

    def step(genome):
        out = ctx.measure(genome)
        if out.status != capi.MEASURED:
            raise SystemExit(f"step failed: status {capi.STATUS_NAMES[out.status]}: {ctx._lib.mmx_last_error(ctx._h).decode()}")
        return out

    for _ in range(max(3, args.warmup)):
        step(GENOME_ALL_NESTS)
    # every step rewrites a, b, c, bt: 4 x N^2 x E = 512 MiB at N=4096 FP64, larger than the 126 MB L2,
    # so no explicit flush is needed between steps
    sampler = ClockSampler(local_rank)
    sampler.start()
    barrier()
    t0 = time.perf_counter()
    device_s = 0.0
    for _ in range(args.steps):
        out = step(GENOME_ALL_NESTS)
        device_s += out.time_s                      # CUDA-event time of the whole individual
    barrier()
    wall_s = time.perf_counter() - t0
    checksum = ctx.stats().checksum
    wall_s = max_over_ranks(wall_s)
    device_s = max_over_ranks(device_s)

    # a genome whose operand is produced on the host: the planner moves `a` up once per step
    mixed = None
    if rank == 0:
        pm = capi.plan(GENOME_MIXED, n, dtype)
        for _ in range(2):
            step(GENOME_MIXED)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        reps = max(3, args.steps // 4)
        for _ in range(reps):
            step(GENOME_MIXED)
        torch.cuda.synchronize()
        mixed = {"genome": GENOME_MIXED, "value": flops * reps / (time.perf_counter() - t1) / 1e9, "unit": "GFLOP/s",
                 "h2d_bytes_per_step": int(pm.h2d_bytes), "d2h_bytes_per_step": int(pm.d2h_bytes),
                 "note": "init-a runs on one host core inside the timed region, then a (N^2 E bytes) is copied from pinned memory"}

    # the contraction as an offload from HOST buffers (the paper's per-region copy pattern made explicit): a, bt, c go up
    # from pinned memory, gene 8 runs, c comes back -- all through the C ABI, inside the timed region
    host_io = None
    if rank == 0:
        host_io = e2e_host_buffers(ctx, n, dtype, esz, max(3, args.steps // 20))

    # roofline of the dominant kernel, measured live (CUDA events on the library's stream, L2 flushed)
    roof = hbm_roof = None
    if rank == 0:
        peaks, peaks_kind = load_measured_peaks()
        ms8 = ctx.time_loop(8, 5, True)
        ach = flops / (ms8 * 1e-3) / 1e12
        share_ms8 = ms8 * 1e-3 / (device_s / args.steps)
        form = ctx.gene8_form() if dtype == capi.F64 else -1
        if form > 0:
            # auto mode picked an INT8 tensor-core form on the device (mmx_gene8_form: 100 SA + 10 SB + levels): digits a_1..a_SA
            # against b_1..b_SB, pairs kept up to level t + u <= levels + 1.  This workload's operands carry log2(N) + 2 bits =
            # two 8-bit digits each up to N = 16384: the 2 x 2 form, 4 INT8 slice products per FP64 term.  ms8 covers the two
            # slice passes, that contraction and the guarded FP64-pipe launch that exits at once.
            sa, sb, lv = form // 100, form // 10 % 10, form % 10
            products = sum(1 for t in range(1, sa + 1) for u in range(1, sb + 1) if t + u <= lv + 1)
            int8_inferred = 2.0 * peaks["bf16_tflops"]
            int8_peak = capi.peak_probe(capi.PEAK_UMMA_I8, local_rank)     # measured in this run (csrc/peaks.cu)
            # the dominant kernel by itself: the contraction launch (plus the guarded FP64-pipe launch that retires at once)
            # on operands encoded once -- mmx_time_gene8_contraction; then the whole nest as the step runs it
            msk = ctx.time_gene8_contraction(5, True)
            ops = products * flops / (msk * 1e-3) / 1e12
            ops_nest = products * flops / (ms8 * 1e-3) / 1e12
            roof = {"bound": "tensor", "pipe": "int8 (tcgen05.mma.kind::i8, INT32 accumulators in TMEM)",
                    "kernel": f"matmul_ozaki_auto form {form} (gene 8 contraction: exact 8-bit INT8 digit slices, {sa} x {sb} digit pairs = {products} "
                              f"slice products per FP64 term)",
                    "form": form, "slice_products_per_term": products,
                    "achieved": ops, "peak": int8_peak, "unit": "TOP/s", "frac": ops / int8_peak,
                    "peak_inferred": int8_inferred, "frac_vs_inferred": ops / int8_inferred,
                    "traffic": ncu_traffic("matmul_ozaki_auto_pair", n) or ncu_traffic("matmul_ozaki_auto", n), "ms_per_launch": msk, "share_of_step": msk * 1e-3 / (device_s / args.steps),
                    "effective_fp64_tflops": flops / (msk * 1e-3) / 1e12,
                    "nest_standalone": {"what": "gene 8 launched by itself (mmx_time_loop): its own two slice passes + the contraction + the guarded "
                                                "FP64-pipe launch -- what a genome pays whose a / bt do not come from the device's fill / transpose "
                                                "kernels; in the timed step those kernels write the digit planes and gene 8 is the contraction alone",
                                        "ms": ms8, "achieved": ops_nest, "frac": ops_nest / int8_peak,
                                        "effective_fp64_tflops": ach,
                                        "vs_fp64_pipe_peak": ach / capi.peak_probe(capi.PEAK_FP64_FMA, local_rank)},
                    "peak_source": "tcgen05.mma.kind::i8 issue peak measured in this run by csrc/peaks.cu (M=128 x N=256 instructions back to back "
                                   "on operands resident in shared memory, one issuing thread per SM); peak_inferred = twice "
                                   "MEASURED_PEAKS.json bf16_tflops (cuBLAS bf16, loads included); achieved counts the INT8 slice products "
                                   "issued per FP64 term (algorithmic work of this form: products x 2N^3)"}
        else:
            pipe_peak = capi.peak_probe(capi.PEAK_FP64_FMA if dtype == capi.F64 else capi.PEAK_FP32_FMA, local_rank)
            roof = {"bound": "tensor", "pipe": "fp64 (DMMA.8x8x4 via mma.sync)" if dtype == capi.F64 else "fp32 (FFMA)",
                    "kernel": "matmul_nt (gene 8)", "achieved": ach, "peak": pipe_peak, "unit": "TFLOP/s", "frac": ach / pipe_peak,
                    "traffic": ncu_traffic("matmul_dmma" if dtype == capi.F64 else "matmul_3xtf32s", n), "ms_per_launch": ms8,
                    "share_of_step": share_ms8,
                    "peak_source": "FMA-issue peak of the same pipe measured in this run by csrc/peaks.cu "
                                   "(MEASURED_PEAKS.json carries only HBM and bf16 figures)"}
        ms6 = ctx.time_loop(6, 10, True)
        gb = 2.0 * esz * n * n / (ms6 * 1e-3) / 1e9
        hbm_roof = {"bound": "hbm", "kernel": "transpose_tiled (gene 6)", "achieved": gb, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gb / peaks["hbm_gbs"], "traffic": ncu_traffic("transpose_tile", n),
                    "peak_source": f"MEASURED_PEAKS.json ({peaks_kind})"}

    # FP32 arm of the same configuration (BASELINE configs[1] names both precisions): whole individuals through
    # the C ABI, then the gene-8 kernel alone (tcgen05 split-TF32 with compensated accumulation, matmul_tc.cu)
    fp32 = None
    if rank == 0 and dtype == capi.F64 and not args.no_fp32:
        fp32 = fp32_arm(n, local_rank, max(10, args.steps // 4), peaks)

    # the same configuration with gene 8 forced onto the FP64 pipe (matmul_variant 4: DMMA), for comparison
    fp64_pipe = None
    if rank == 0 and dtype == capi.F64 and n >= 1024 and not args.no_fp64_pipe:
        fp64_pipe = fp64_pipe_arm(n, local_rank, max(10, args.steps // 4), checksum)

    # the same configuration on operands WITHOUT the application's special structure (SURVEY 8d config 2's optional run)
    fp64_random = None
    if rank == 0 and dtype == capi.F64 and n >= 1024 and not args.no_fp64_random:
        fp64_random = fp64_random_arm(n, local_rank)

    # the sampler covers the timed region plus the (equally loaded) mixed-genome and roofline phases
    clocks = sampler.stop()

    # >= 3 s of individuals back to back, then ~2 s of the dominant kernel back to back: the numbers above are burst-clock figures
    sustained = None
    if rank == 0 and not args.no_sustained:
        sustained = sustained_block(ctx, n, dtype, local_rank, roof, args.sustained_seconds)

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(n, 0 if dtype == capi.F64 else 1, os.cpu_count() or 1)

    line = None
    if rank == 0:
        ms_per_step = 1e3 * wall_s / args.steps
        line = {
            "metric": "matrix_app_gflops", "value": flops * args.steps * world / device_s / 1e9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "dtype_note": ("operands, results and every kernel but gene 8 are f64; gene 8 multiplies exact int8 digits of the f64 operands "
                           "on the tensor cores (int32 sums) and rebuilds the f64 result, bit-identical to the f64 pipe here; the "
                           "fp64_pipe arm is the same run without that" if (dtype == capi.F64 and n >= 1024) else None),
            "data": "synthetic (the program generates its own inputs: a=(i+j)/N, b=(i-j)/N)",
            "config": {"workload": f"matrix app N={n} {args.dtype}, genome {GENOME_ALL_NESTS} (all six loop nests offloaded)",
                       "gene8": ("auto: INT8 tensor cores in the cheapest error-free form, chosen on the device from the operands "
                                 f"(form {roof.get('form')} here), FP64 pipe otherwise"
                                 if (dtype == capi.F64 and n >= 1024 and roof) else "default kernel for this dtype and size"),
                       "n": n, "genome": GENOME_ALL_NESTS, "individuals_per_step_per_gpu": 1,
                       "l2": "working set 4*N^2*E per step exceeds L2; no flush needed"},
            "e2e": {"value": flops * args.steps * world / wall_s / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(plan.h2d_bytes), "d2h_bytes_per_step": int(plan.d2h_bytes),
                    "note": "host clock around mmx_measure (plan + 6 launches + checksum D2H + sync); this genome has no host-side inputs"},
            "e2e_mixed": mixed, "e2e_host_buffers": host_io,
            # the plan counts one launch per offloaded nest.  In auto mode at N % 64 == 0 (N >= 1024) a captured individual is six
            # kernels: init-a (+ digit planes), the column exponents of b (what is left of the init-b step), zero-c, the transpose
            # (computes its tiles of b, writes b, bt + digit planes), the tensor-core contraction, the trace -- the fallback of auto
            # mode sits in a conditional graph node that does not run (profiles/*_launches.csv lists the un-captured form, where a
            # guarded FP64-pipe launch retires at once: seven)
            "gpu_launches": (int(plan.kernel_launches) + (0 if (n >= 1024 and n % 64 == 0) else
                                                          3 if (dtype == capi.F64 and n >= 1024) else 0)) * args.steps,
            "clocks": clocks, "roofline": roof, "roofline_hbm": hbm_roof, "cpu_baseline": base,
            "checksum": checksum,
        }
        if fp32 is not None:
            line["fp32"] = fp32
        if fp64_pipe is not None:
            line["fp64_pipe"] = fp64_pipe
        if fp64_random is not None:
            line["fp64_random"] = fp64_random
        if sustained is not None:
            line["sustained"] = sustained

    # config 4 / config 5 (every rank takes part): the GA search with the population sharded over the ranks, and the row-sharded
    # individual with the fused transpose + exchange over peer memory.  The line above is complete before they start: a block that
    # raises is reported as {"error": ...}, and a block that does not return within --multi-budget seconds (a member lost while its
    # peers wait on its events) makes rank 0 print the line with that error and every rank leave -- the headline never depends on them
    if (world > 1 and not args.no_multi) or args.ga:
        import threading

        import signal
        gave_up = threading.Lock()

        def give_up(why=None):
            if not gave_up.acquire(blocking=False):
                return
            if rank == 0:
                line["multi_gpu"] = {"error": why or f"the multi-GPU blocks did not return within {args.multi_budget:.0f} s; abandoned"}
                print(json.dumps(line), flush=True)
            os._exit(0)

        watchdog = threading.Timer(args.multi_budget, give_up)
        watchdog.daemon = True
        watchdog.start()
        # a rank that dies hard makes the launcher SIGTERM the others: rank 0 still prints its line.  The main thread may sit inside a
        # C call (a CUDA synchronise, a gloo collective) where Python-level handlers do not run, so the signal is taken from the wakeup
        # pipe by a watcher thread
        wake_r, wake_w = os.pipe()
        os.set_blocking(wake_w, False)
        signal.signal(signal.SIGTERM, lambda *_: None)
        signal.set_wakeup_fd(wake_w, warn_on_full_buffer=False)

        def on_sigterm():
            os.read(wake_r, 1)
            give_up("terminated by the launcher while the multi-GPU blocks ran (another rank died)")

        threading.Thread(target=on_sigterm, daemon=True).start()
        multi = {}
        try:
            multi["ga"] = ga_block(args, n, dtype, device, rank, world, ctl, barrier)
        except Exception as e:  # noqa: BLE001 -- reported in the line, never fatal for it
            multi["ga"] = {"error": f"{type(e).__name__}: {e}"}
        if world > 1:
            try:
                multi["rowshard"] = rowshard_block(args, dtype, device, rank, world, ctl, max_over_ranks, barrier)
            except Exception as e:  # noqa: BLE001
                multi["rowshard"] = {"error": f"{type(e).__name__}: {e}"}
        else:
            multi["rowshard"] = {"skipped": "needs --gpus >= 2 (one process per GPU under torchrun)"}
        watchdog.cancel()
        signal.set_wakeup_fd(-1)
        signal.signal(signal.SIGTERM, signal.SIG_DFL)
        if rank == 0:
            line["multi_gpu"] = multi
        if any(isinstance(v, dict) and "error" in v for v in multi.values()):
            # the ranks may no longer agree on which collective comes next: print and leave without another one
            if rank == 0:
                print(json.dumps(line), flush=True)
            os._exit(0)
    if rank == 0:
        print(json.dumps(line), flush=True)
    try:
        ctx.close()
    except Exception:  # noqa: BLE001 -- a device a failed block left unusable must not turn a printed line into a non-zero exit
        pass
    if world > 1:
        dist.destroy_process_group()


def e2e_host_buffers(ctx, n, dtype, esz, reps):
    import numpy as np
    import torch

    from paper_1806_01430_b200 import capi
    tdt = torch.float64 if dtype == capi.F64 else torch.float32
    i = torch.arange(n, dtype=tdt)
    pinned = {capi.ARRAY_A: ((i[:, None] + i[None, :]) / n).pin_memory(), capi.ARRAY_BT: ((i[None, :] - i[:, None]) / n).pin_memory(),
              capi.ARRAY_C: torch.zeros((n, n), dtype=tdt).pin_memory()}
    out = torch.empty((n, n), dtype=tdt).pin_memory()
    lib, h = ctx._lib, ctx._h

    def once():
        for arr, t in pinned.items():
            ctx._check(lib.mmx_upload_array(h, 0, arr, t.data_ptr(), t.numel() * esz))
        ctx.run_loop(8)
        ctx._check(lib.mmx_fetch_array(h, 0, capi.ARRAY_C, out.data_ptr(), out.numel() * esz))

    once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        once()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    # closed form of the application's product: c[0][0] = S2 / N^2
    s2 = (n - 1) * n * (2 * n - 1) / 6
    ok = bool(np.isclose(float(out[0, 0]), s2 / (n * n), rtol=1e-5 if dtype == capi.F32 else 1e-12))
    return {"value": 2.0 * n ** 3 / dt / 1e9, "unit": "GFLOP/s", "ms_per_step": dt * 1e3, "h2d_bytes_per_step": 3 * n * n * esz,
            "d2h_bytes_per_step": n * n * esz, "result_checked": ok,
            "note": "mmx_upload_array x3 (pinned host -> device) + gene-8 kernel + mmx_fetch_array of c (device -> pinned host), host clock"}


def fp64_random_arm(n, device):
    """Gene 8 on uniform(-1, 1) operands from MT19937(seed 1) -- NOT the reference's inputs (the program generates its own): full
    53-bit mantissas, so no INT8 digit form is error-free and auto mode takes the FP64 pipe (DMMA).  Beside it the opt-in general
    tensor-core kernel (matmul_variant 40: 7 exact 8-bit slices per operand, 28 slice products per term, truncation bound
    2e-14 K max|a| max|b|), with its measured norm-wise error on a sample of rows."""
    import numpy as np

    from paper_1806_01430_b200 import capi
    rng = np.random.Generator(np.random.MT19937(1))
    a = rng.uniform(-1.0, 1.0, (n, n))
    b = rng.uniform(-1.0, 1.0, (n, n))
    flops = 2.0 * n ** 3
    rows = np.arange(0, n, max(1, n // 16))[:16]
    exact = a[rows] @ b                                  # float64 dot of the sampled rows (host; 16 rows only)
    bound = np.abs(a[rows]) @ np.abs(b)                  # sum_k |a_ik| |b_kj|: the norm-wise bar's scale
    out = {"data": "uniform(-1,1), numpy MT19937 seed 1 (non-reference inputs)"}
    for label, variant in (("auto", 0), ("int8_7_slices", 40)):
        with capi.Context(n=n, dtype=capi.F64, devices=[device], matmul_variant=variant, timeout_s=600.0) as ctx:
            ctx.upload(capi.ARRAY_A, a)
            ctx.upload(capi.ARRAY_B, b)
            ctx.run_loop(4)
            ctx.run_loop(6)
            ctx.run_loop(8)
            c = ctx.fetch(capi.ARRAY_C)[rows]
            err = float((np.abs(c - exact) / bound).max())
            ms8 = ctx.time_loop(8, 3, True)
            form = ctx.gene8_form() if variant == 0 else 777
            pipe_peak = capi.peak_probe(capi.PEAK_FP64_FMA, device)
        out[label] = {"gene8_form": form, "ms_per_launch": ms8, "effective_fp64_tflops": flops / ms8 / 1e9,
                      "vs_fp64_pipe_peak": flops / ms8 / 1e9 / pipe_peak, "max_normwise_error": err, "tolerance": 1e-12,
                      "kernel": ("matmul_dmma on the FP64 pipe (auto mode found no error-free INT8 form: gene8_form 0); slice passes and the "
                                 "auto launch that retires at once included" if variant == 0 else
                                 "matmul_ozaki fixed 7-slice triangular form on the INT8 tensor cores (opt-in: its bound is relative to "
                                 "the row maxima, not to sum|a||b|, so auto mode does not take it)")}
    return out


def sustained_block(ctx, n, dtype, device, roof, seconds):
    """The timed region of the headline is milliseconds long (burst clocks).  Here: individuals back to back for >= `seconds`, clocks
    sampled, then the dominant kernel back to back for ~2 s inside one event pair (mmx_time_gene8_contraction, flush_l2 = 2)."""
    from paper_1806_01430_b200 import capi
    flops = 2.0 * n ** 3
    sampler = ClockSampler(device)
    sampler.start()
    t0 = time.perf_counter()
    dev_s, k = 0.0, 0
    while time.perf_counter() - t0 < seconds:
        for _ in range(50):
            dev_s += ctx.measure(GENOME_ALL_NESTS).time_s
        k += 50
    wall = time.perf_counter() - t0
    clocks_ind = sampler.stop()
    out = {"individuals": k, "wall_s": wall, "value": flops * k / dev_s / 1e9, "e2e": flops * k / wall / 1e9, "unit": "GFLOP/s",
           "ms_per_individual": 1e3 * dev_s / k, "clocks": clocks_ind}
    if roof is not None and roof.get("form"):
        iters = max(100, int(2.0 / (roof["ms_per_launch"] * 1e-3)))
        sampler = ClockSampler(device)
        sampler.start()
        ms = ctx.time_gene8_contraction(iters, 2)
        clocks_k = sampler.stop()
        ops = roof["slice_products_per_term"] * flops / (ms * 1e-3) / 1e12
        scale = (clocks_k["sm_mhz"] / clocks_k["sm_max_mhz"]) if clocks_k.get("sm_mhz") and clocks_k.get("sm_max_mhz") else None
        out["contraction"] = {"launches": iters, "ms_per_launch": ms, "achieved": ops, "unit": "TOP/s", "peak": roof["peak"],
                              "frac": ops / roof["peak"], "clocks": clocks_k,
                              "frac_at_the_sampled_clock": ops / (roof["peak"] * scale) if scale else None,
                              "note": "back to back inside one CUDA-event pair, operands encoded once; peak = the burst issue peak of "
                                      "roofline.peak, frac_at_the_sampled_clock scales it by median SM clock / max SM clock"}
    return out


def ncu_traffic(kernel: str, n: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the committed `ncu --set full`
    summary (profiles/ncu_traffic.json, written by tools/ncu_summary.py --traffic); None when not captured at this N."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        table = json.loads(p.read_text())
    except (OSError, ValueError):
        return None
    hit = table.get(f"{kernel}@{n}")
    return hit["bytes_per_launch"] if hit else None


def fp32_arm(n, device, steps, peaks):
    """FP32 arm of the same configuration, plus the same steps with gene 8 forced onto the split-TF32 kernel (variant 30: what
    operands without a short exact digit form get)."""
    from paper_1806_01430_b200 import capi
    flops = 2.0 * n ** 3

    def run(variant):
        with capi.Context(n=n, dtype=capi.F32, devices=[device], timeout_s=600.0, matmul_variant=variant) as ctx:
            for _ in range(3):
                ctx.measure(GENOME_ALL_NESTS)
            dev_s = 0.0
            t0 = time.perf_counter()
            for _ in range(steps):
                dev_s += ctx.measure(GENOME_ALL_NESTS).time_s
            wall = time.perf_counter() - t0
            return dev_s, wall, ctx.time_loop(8, 5, True), ctx.gene8_form()

    dev_s, wall, ms8, form = run(0)
    ffma_peak = capi.peak_probe(capi.PEAK_FP32_FMA, device)
    out = {"dtype_note": "FP32 parity is against the EXACT product of the float operands (norm-wise 1e-6 bar, SURVEY H2 option i), not against "
                         "the CPU float program: where an INT8 form applies c is that product rounded once to float, which differs from the "
                         "reference's own float output (k-ascending float accumulation, ~1e-3 element-wise at N >= 1024) because the reference "
                         "is the less accurate of the two; MMX_NUMERICS_STRICT reproduces the CPU float program bit for bit",
           "value": flops * steps / dev_s / 1e9, "unit": "GFLOP/s", "steps": steps, "e2e": flops * steps / wall / 1e9,
           "ms_per_launch": ms8, "effective_fp32_tflops": flops / ms8 / 1e9,
           "vs_ffma_pipe_peak": flops / ms8 / 1e9 / ffma_peak, "ffma_pipe_peak_tflops": ffma_peak}
    tf32_inferred = peaks["bf16_tflops"] / 2.0
    tf32_peak = capi.peak_probe(capi.PEAK_UMMA_TF32, device)

    def tf32_roof(ms):
        return {"bound": "tensor", "achieved": 3.0 * flops / ms / 1e9, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": 3.0 * flops / ms / 1e9 / tf32_peak, "peak_inferred": tf32_inferred,
                "frac_vs_inferred": 3.0 * flops / ms / 1e9 / tf32_inferred, "traffic": ncu_traffic("matmul_3xtf32s", n),
                "peak_source": "tcgen05.mma.kind::tf32 issue peak measured in this run (csrc/peaks.cu); peak_inferred = half of "
                               "MEASURED_PEAKS.json bf16_tflops; achieved counts the three tensor-core products issued per FP32 term"}
    tf32_kernel = ("matmul_3xtf32s (gene 8: three TF32 products per term on tcgen05, b parts stacked along N so two of them share one "
                   "N=256 MMA; compensated accumulation; split passes included)")
    if form > 0:
        sa, sb, lv = form // 100, form // 10 % 10, form % 10
        products = sum(1 for t in range(1, sa + 1) for u in range(1, sb + 1) if t + u <= lv + 1)
        int8_inferred = 2.0 * peaks["bf16_tflops"]
        int8_peak = capi.peak_probe(capi.PEAK_UMMA_I8, device)
        ops = products * flops / ms8 / 1e9
        out["kernel"] = (f"matmul_ozaki_auto<float> form {form} (gene 8: the float operands' exact 8-bit INT8 digits, {sa} x {sb} pairs = "
                         f"{products} slice products per term, result = the exact product rounded once to float; slice passes and the "
                         f"three guarded split-TF32 launches included)")
        out["roofline"] = {"bound": "tensor", "pipe": "int8", "achieved": ops, "peak": int8_peak, "unit": "TOP/s", "frac": ops / int8_peak,
                           "peak_inferred": int8_inferred, "frac_vs_inferred": ops / int8_inferred,
                           "traffic": None, "form": form, "slice_products_per_term": products,
                           "peak_source": "tcgen05.mma.kind::i8 issue peak measured in this run (csrc/peaks.cu); whole nest (digit planes included)"}
        d2, w2, ms30, _ = run(30)
        out["split_tf32"] = {"value": flops * steps / d2 / 1e9, "unit": "GFLOP/s", "e2e": flops * steps / w2 / 1e9, "kernel": tf32_kernel,
                             "ms_per_launch": ms30, "effective_fp32_tflops": flops / ms30 / 1e9, "roofline": tf32_roof(ms30),
                             "note": "the same steps with matmul_variant 30: what gene 8 runs when no INT8 form is error-free"}
    else:
        out["kernel"] = tf32_kernel
        out["roofline"] = tf32_roof(ms8)
    return out


def fp64_pipe_arm(n, device, steps, reference_checksum):
    """The same steps with gene 8 on the FP64 pipe (DMMA).  Results are bit-identical to the default path on this workload
    (checked here on c's corners and the checksum; tests compare all of c)."""
    from paper_1806_01430_b200 import capi
    flops = 2.0 * n ** 3
    with capi.Context(n=n, dtype=capi.F64, matmul_variant=4, devices=[device], timeout_s=600.0) as ctx:
        for _ in range(3):
            ctx.measure(GENOME_ALL_NESTS)
        dev_s = 0.0
        t0 = time.perf_counter()
        for _ in range(steps):
            dev_s += ctx.measure(GENOME_ALL_NESTS).time_s
        wall = time.perf_counter() - t0
        checksum = ctx.stats().checksum
        c = ctx.fetch(capi.ARRAY_C)
        ms8 = ctx.time_loop(8, 5, True)
        pipe_peak = capi.peak_probe(capi.PEAK_FP64_FMA, device)
    s2 = (n - 1) * n * (2 * n - 1) / 6
    ach = flops / ms8 / 1e9
    return {"value": flops * steps / dev_s / 1e9, "unit": "GFLOP/s", "steps": steps, "e2e": flops * steps / wall / 1e9,
            "kernel": "matmul_dmma (gene 8: mma.sync.m8n8k4.f64, 64x64 tiles, 3 CTAs per SM)", "ms_per_launch": ms8,
            "bit_identical_to_default_path": bool(checksum == reference_checksum and float(c[0, 0]) == s2 / (n * n)
                                                  and float(c[1, 2]) == (s2 - n * (n - 1) / 2 - 2 * n) / (n * n)),
            "roofline": {"bound": "tensor", "pipe": "fp64 (DMMA.8x8x4 via mma.sync)", "achieved": ach, "peak": pipe_peak, "unit": "TFLOP/s",
                         "frac": ach / pipe_peak, "traffic": ncu_traffic("matmul_dmma", n),
                         "peak_source": "FMA-issue peak of the FP64 pipe measured in this run by csrc/peaks.cu"}}


def ga_block(args, n, dtype, device, rank, world, ctl, barrier):
    """BASELINE config 4: GA 64 x 40, seed 1, real CUDA-event fitness at N=4096, population sharded over the ranks
    (sharded.ShardedEvaluator: every rank walks the same GA, measures its share of each generation's unseen genomes on its own GPU,
    outcomes gathered as 4 doubles per genome over gloo -- the pool semantics of evaluator.cpp:246-276 across processes)."""
    import torch.distributed as dist

    from paper_1806_01430_b200 import capi
    from paper_1806_01430_b200.sharded import ShardedEvaluator
    cores = os.cpu_count() or 1
    team = max(1, cores // world)                 # host threads for CPU-mapped nests: the ranks share the box's cores
    zero = "0" * capi.GENE_LENGTH
    # the all-CPU baseline genome must be MEASURED (ga.cpp:254-258); at N=4096 it takes seconds even on every core, so it is measured
    # once, on rank 0, on all cores, outside the search (budget 300 s) and preloaded like a line of eval_cache.jsonl
    base = [None]
    t_base = time.perf_counter()
    if rank == 0:
        with capi.Context(n=n, dtype=dtype, devices=[device], timeout_s=300.0, host_threads=cores) as bctx:
            base[0] = bctx.measure(zero).as_tuple()
    if world > 1:
        dist.broadcast_object_list(base, src=0, group=ctl)
    t_base = time.perf_counter() - t_base
    if base[0][0] != capi.MEASURED:
        return {"skipped": f"the all-CPU baseline genome could not be measured within 300 s (status {capi.STATUS_NAMES[base[0][0]]})"}
    # each rank's CPU-mapped nests run on the rank's own share of the host's CPUs (mmx_config.pin_host)
    with capi.Context(n=n, dtype=dtype, devices=[device], timeout_s=args.ga_timeout, host_threads=team,
                      host_core_first=(rank % max(1, cores // team)) * team, host_core_count=team,
                      early_timeout=0 if args.ga_wait_timeouts else 1) as ctx:
        ev = ShardedEvaluator(lambda g: ctx.measure(g).as_tuple(), capi.GENE_LENGTH, group=ctl, device="cpu")
        ev.preload(zero, base[0])
        barrier()
        t0 = time.perf_counter()
        res = ev.run_ga(population=args.ga_population, generations=args.ga_generations, seed=1)
        barrier()
        wall = time.perf_counter() - t0
        c = ev.counters()
        local = ev.local_measurements
        walls = list(ev.batch_wall)
    rows = res["csv"].splitlines()[1:]
    first_best = next(int(r.split(",")[0]) for r in rows if r.split(",")[3] == res["best_genome"])
    feasible = sum(1 for o in ev.memo.values() if o[0] != capi.COMPILE_ERROR)
    timeouts = sum(1 for o in ev.memo.values() if o[0] == capi.TIMEOUT)
    per_rank = [local]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, local, group=ctl)
    out = {"config": f"GA {args.ga_population} x {args.ga_generations}, seed 1, N={n}, budget {args.ga_timeout} s per individual, "
                     f"{team} host thread(s) per rank for CPU-mapped nests",
           "early_timeout": not args.ga_wait_timeouts,
           "wall_s": wall, "wall_to_best_s": walls[first_best] - (walls[0] if walls else 0.0) if first_best < len(walls) else None,
           "generation_of_best": first_best, "best_genome": res["best_genome"], "best_s": res["best_s"],
           "baseline_s": res["baseline_s"], "baseline_measure_s": t_base,
           "speedup_vs_all_cpu_genome": res["baseline_s"] / res["best_s"],
           "requests": c["requests"], "distinct": c["distinct"], "cache_hits": c["cache_hits"],
           "feasible_measured": feasible, "timeouts": timeouts, "measured_per_rank": per_rank,
           "individuals_per_s": c["distinct"] / wall, "feasible_individuals_per_s": feasible / wall,
           "paper_budget_fraction": (wall + t_base) / 3600.0,
           "note": "wall_s covers the whole search (2522 requests); infeasible genomes are rejected by the planner without GPU work; "
                   "genomes that leave the matmul nest on the host cannot meet the budget and score it (evaluator.cpp:103-108) -- with "
                   "early_timeout such a run is given up as soon as its measured progress shows that (same outcome, a fraction of the wall cost)"}
    out["key"] = [n, args.ga_population, args.ga_generations, args.ga_timeout, not args.ga_wait_timeouts]
    try:   # the same block measured on ONE GPU (committed evidence: bench.py --ga on one B200), for the efficiency figure
        one = json.loads((ROOT / "profiles" / "r2_ga_n1.json").read_text())
        if world > 1 and one.get("key") == out["key"]:
            out["n1_wall_s"] = one["wall_s"]
            out["speedup_vs_n1"] = one["wall_s"] / wall
            out["efficiency_vs_n1"] = one["wall_s"] / wall / world
            out["n1_source"] = "profiles/r2_ga_n1.json"
    except (OSError, ValueError, KeyError):
        pass
    return out


def rowshard_block(args, dtype, device, rank, world, ctl, max_over_ranks, barrier):
    """BASELINE config 5: one individual row-sharded over the ranks (rowshard.RowShardedRun over mmx_shard_*): the transpose stores
    its rows of bt into every member's bt through peer-mapped pointers (the exchange IS the transpose kernel), the contraction walks
    the column blocks in ring order gated by the owners' events.  Per N: TFLOP/s of the sharded individual (max gpu_ms over the
    ranks), the single-GPU individual on rank 0 for comparison, the exchange against the 900 GB/s per direction NVLink 5 bound."""
    import torch

    from paper_1806_01430_b200 import capi
    from paper_1806_01430_b200.rowshard import GpuMember, RowShardedRun
    esz = 8 if dtype == capi.F64 else 4
    out = []
    if os.environ.get("MMX_BENCH_INJECT") == f"rowshard_raise_{rank}":   # test hook: this rank fails, its peers are left waiting
        raise RuntimeError("injected failure (MMX_BENCH_INJECT)")
    if os.environ.get("MMX_BENCH_INJECT") == f"rowshard_die_{rank}":     # test hook: this rank dies hard, the launcher ends the others
        os._exit(3)
    for n in args.rowshard_n:
        flops = 2.0 * n ** 3
        need = 4 * n * n * esz + 15 * n * n + (1 << 30)       # arrays + digit planes + slack
        free, _total = torch.cuda.mem_get_info(device)
        share = os.environ.get("MMX_BENCH_SHARE_DEVICE") == "1"
        ok = max_over_ranks(1.0 if need * (world if share else 1) > free else 0.0) == 0.0
        if not ok:
            out.append({"n": n, "skipped": f"needs {need / 2**30:.0f} GiB per member, {free / 2**30:.0f} GiB free"})
            continue
        with capi.Context(n=n, dtype=dtype, devices=[device], timeout_s=600.0) as ctx:
            run = RowShardedRun(GpuMember(ctx), ctl, dtype == capi.F32)
            run.run()                                           # warm-up (first-use work, graph-free path)
            reps = 3
            barrier()
            t0 = time.perf_counter()
            rs = [run.run() for _ in range(reps)]
            barrier()
            wall = (time.perf_counter() - t0) / reps
            gpu_ms = max_over_ranks(sum(r["gpu_ms"] for r in rs) / reps)
            x_ms = max_over_ranks(sum(r["exchange_ms"] for r in rs) / reps)
            mm_ms = max_over_ranks(sum(r["matmul_ms"] for r in rs) / reps)
            peer_bytes = rs[-1]["peer_bytes"]
            checksum = rs[-1]["checksum"]
            barrier()
            single = None
            if rank == 0:                                       # the same individual on one GPU, same context
                ctx.measure(GENOME_ALL_NESTS)
                o = ctx.measure(GENOME_ALL_NESTS)
                single = {"ms": o.time_s * 1e3, "tflops": flops / o.time_s / 1e12, "checksum": ctx.stats().checksum}
            barrier()
        row = {"n": n, "world": world, "ms": gpu_ms, "tflops": flops / (gpu_ms * 1e-3) / 1e12, "wall_ms": wall * 1e3,
               "exchange_ms": x_ms, "matmul_ms": mm_ms, "peer_bytes_per_member": peer_bytes,
               "exchange_gbs_per_member": peer_bytes / (x_ms * 1e-3) / 1e9 if x_ms > 0 else None,
               "exchange_frac_of_nvlink": peer_bytes / (x_ms * 1e-3) / 1e9 / 900.0 if x_ms > 0 else None,
               "nvlink_peak_gbs_per_direction": 900.0, "checksum": checksum, "single_gpu": single}
        if single is not None:
            row["speedup_vs_single_gpu"] = single["ms"] / gpu_ms
            row["frac_of_n_x_single_gpu"] = single["ms"] / gpu_ms / world
        if share:
            row["note"] = "MMX_BENCH_SHARE_DEVICE=1: all members on ONE device (peer stores are local stores); not a scaling number"
        out.append(row)
    return out


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
