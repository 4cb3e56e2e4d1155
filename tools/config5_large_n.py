#!/usr/bin/env python
"""BASELINE config 5: large-N sweep.  Per N: the gene-8 kernel alone (FP64 and FP32), the whole all-nests individual, and the
row-sharded individual over `world` slots.  On a one-GPU box the slots share the device, so the sharded numbers show only
the overhead of the fused transpose+all-gather and of the column-block contraction, not a speed-up; on an 8-GPU box pass
--devices 0 1 ... to spread the members.  python tools/config5_large_n.py --n 4096 8192 16384 32768 --world 1 2 4"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[4096, 8192, 16384])
ap.add_argument("--world", type=int, nargs="+", default=[1, 2, 4])
ap.add_argument("--devices", type=int, nargs="*", default=None)
ap.add_argument("--dtypes", nargs="+", default=["f64", "f32"])
args = ap.parse_args()

for n in args.n:
    for name in args.dtypes:
        dtype, e = (capi.F64, 8) if name == "f64" else (capi.F32, 4)
        flops = 2.0 * n ** 3
        with capi.Context(n=n, dtype=dtype, timeout_s=600.0) as ctx:
            out = ctx.measure("101010101001")
            out = ctx.measure("101010101001")
            ms8 = ctx.time_loop(8, 2 if n >= 16384 else 4, True)
            print(json.dumps({"n": n, "dtype": name, "what": "single GPU", "individual_ms": out.time_s * 1e3,
                              "app_tflops": flops / out.time_s / 1e12, "matmul_ms": ms8, "matmul_tflops": flops / ms8 / 1e9,
                              "checksum": ctx.stats().checksum}), flush=True)
        for world in args.world:
            if 4 * world * n * n * e > 150e9:
                continue
            devs = (args.devices[:world] if args.devices else [0] * world)
            with capi.Context(n=n, dtype=dtype, num_slots=world, devices=devs, timeout_s=600.0) as ctx:
                ctx.shard_run_local()
                checksum, stats = ctx.shard_run_local()
                print(json.dumps({"n": n, "dtype": name, "what": f"row-sharded, world {world}, devices {devs}",
                                  "gpu_ms_max": max(s["gpu_ms"] for s in stats), "exchange_ms_max": max(s["exchange_ms"] for s in stats),
                                  "matmul_ms_max": max(s["matmul_ms"] for s in stats), "peer_bytes_per_member": stats[0]["peer_bytes"],
                                  "app_tflops": flops / (max(s["gpu_ms"] for s in stats) * 1e-3) / 1e12, "checksum": checksum}), flush=True)
