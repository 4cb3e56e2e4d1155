"""bench.py under the driver's multi-GPU launch line (torchrun, one process per rank), on whatever GPUs the box has: with one GPU
both ranks share cuda:0 (MMX_BENCH_SHARE_DEVICE=1, gloo instead of NCCL -- NCCL refuses two ranks on one device); with >= 2 GPUs the
contract's own launch runs (NCCL, one device per rank).  Checks that the JSON line carries the config-4 (GA, population sharded) and
config-5 (row-sharded individual over IPC peer memory) blocks and that their results are the right ones."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_bench_two_ranks_reports_ga_and_rowshard_blocks():
    import torch
    world = 2
    env = dict(os.environ)
    if torch.cuda.device_count() < world:
        env["MMX_BENCH_SHARE_DEVICE"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", str(world), "--steps", "5", "--warmup", "3", "--size", "1024",
           "--no-cpu-baseline", "--no-fp32", "--no-fp64-pipe", "--ga-population", "12", "--ga-generations", "4", "--ga-timeout", "1.0",
           "--rowshard-n", "1024", "2048"]
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=540)
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == world and line["value"] > 0 and line["checksum"] == 0.0
    ga = line["multi_gpu"]["ga"]
    assert "skipped" not in ga, ga
    assert ga["requests"] == 1 + 12 + 3 * 11 and ga["best_s"] < ga["baseline_s"]
    assert sum(ga["measured_per_rank"]) == ga["distinct"] and min(ga["measured_per_rank"]) > 0     # both ranks measured their share
    assert all(ch in "01" for ch in ga["best_genome"]) and len(ga["best_genome"]) == 12
    rs = line["multi_gpu"]["rowshard"]
    assert [r["n"] for r in rs] == [1024, 2048]
    for r in rs:
        assert r["checksum"] == 0.0 == r["single_gpu"]["checksum"]      # N = 2^p: the trace is exactly 0
        assert r["peer_bytes_per_member"] == (r["n"] // world) * r["n"] * 8 * (world - 1)
        assert r["ms"] > 0 and r["exchange_ms"] > 0 and r["tflops"] > 0
