"""The N>1 path on CPU: world_size-2 `gloo` run of the rank-sharded population evaluator.

Each rank measures only its share of a generation's unseen genomes (here with the matrix12 cost model
standing in for the GPU), the outcomes are gathered, and both ranks must walk the exact GA trajectory
the single-process reference produces (tests/golden/ga_runs.json)."""
import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out_dir: str):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from paper_1806_01430_b200.sharded import ShardedEvaluator
    dist.init_process_group("gloo", rank=rank, world_size=world)
    times = np.load(GOLDEN / "model_times_matrix12.npy")

    measured = []

    def measure(genome: str):
        measured.append(genome)
        t = float(times[sum(1 << k for k, ch in enumerate(genome) if ch == "1")])
        return (1, 0.0, 0.0) if t < 0 else (0, t, t)

    ev = ShardedEvaluator(measure, 12, cost=lambda g: 1.0 + g.count("1"))
    res = ev.run_ga(population=12, generations=12, seed=1)
    # a second, larger run on the same evaluator keeps using the memo
    res2 = ev.run_ga(population=16, generations=5, crossover_rate=0.0, mutation_rate=0.0, seed=9)
    out = {"csv": res["csv"], "best": res["best_genome"], "csv2": res2["csv"], "local": len(measured),
           "local_unique": len(set(measured)), "counters": ev.counters(), "memo": len(ev.memo)}
    Path(out_dir, f"rank{rank}.json").write_text(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_ranks_share_the_population_and_replay_the_reference_trajectory(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    outs = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(world)]
    golden = json.loads((GOLDEN / "ga_runs.json").read_text())
    run0 = golden[0]
    for o in outs:
        assert o["csv"] == run0["csv"]                     # byte-identical generations.csv on every rank
        assert o["best"] == run0["best_genome"]
        assert o["local"] == o["local_unique"]             # nothing measured twice
    assert outs[0]["counters"] == outs[1]["counters"]
    # every distinct genome was measured exactly once, by exactly one rank, and both ranks worked
    assert outs[0]["local"] + outs[1]["local"] == outs[0]["memo"] == outs[0]["counters"]["backend_calls"]
    assert min(o["local"] for o in outs) >= 0.3 * outs[0]["memo"]
    # the second run is the golden "no crossover, no mutation" trajectory except for the counters, which
    # continue from the first run (the memo is shared): compare the GA columns only
    want = [r.split(",")[:5] for r in golden[-1]["csv"].splitlines()]
    got = [r.split(",")[:5] for r in outs[0]["csv2"].splitlines()]
    assert got == want


def _failing_worker(rank: int, world: int, port: int, out_dir: str):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from paper_1806_01430_b200.sharded import ShardedEvaluator, ShardedMeasureError
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def measure(genome: str):
        if genome == "111100000000":
            raise RuntimeError("device fell over")
        return (0, 1.0 + genome.count("1"), 0.5)

    ev = ShardedEvaluator(measure, 12, cost=lambda g: 1.0)
    batch = ["000000000000", "111100000000", "100000000000", "010000000000"]
    raised = None
    try:
        ev.evaluate_all(batch)
    except ShardedMeasureError as e:
        raised = str(e)
    before = ev.counters()
    ok = ev.evaluate_all([g for g in batch if g != "111100000000"])     # the group is still in step afterwards
    Path(out_dir, f"rank{rank}.json").write_text(json.dumps({"raised": raised, "before": before, "ok": ok, "after": ev.counters()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_a_failing_measurement_raises_on_every_rank_and_leaves_the_group_in_step(tmp_path):
    world = 2
    mp.spawn(_failing_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    outs = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(world)]
    for o in outs:
        assert o["raised"] is not None and "111100000000" in o["raised"]
        assert o["before"]["requests"] == o["before"]["distinct"] == 0       # the failed batch left no trace
        assert [tuple(x) for x in o["ok"]] == [(0, 1.0, 0.5), (0, 2.0, 0.5), (0, 2.0, 0.5)]
        assert o["after"]["distinct"] == 3
    assert sum("device fell over" in o["raised"] for o in outs) == 1         # the owner reports the cause, the other the fact


def test_assignment_is_deterministic_and_balanced():
    sys.path.insert(0, str(ROOT))
    from paper_1806_01430_b200.sharded import assign_lpt, default_cost
    genomes = ["".join("1" if (m >> k) & 1 else "0" for k in range(12)) for m in range(0, 4096, 7)]
    a = assign_lpt(genomes, 8)
    assert a == assign_lpt(list(genomes), 8)
    loads = [sum(default_cost(g) for g, o in zip(genomes, a) if o == r) for r in range(8)]
    assert max(loads) <= 1.2 * (sum(loads) / 8) + 3000   # within one heavy individual of the mean
    assert default_cost("110000000000") == 0.0            # infeasible genomes cost nothing
    assert default_cost("000000000000") > default_cost("101010101001")


def test_single_process_matches_the_cpp_evaluator():
    sys.path.insert(0, str(ROOT))
    from paper_1806_01430_b200.sharded import ShardedEvaluator
    times = np.load(GOLDEN / "model_times_separable.npy")

    def measure(genome):
        t = float(times[sum(1 << k for k, ch in enumerate(genome) if ch == "1")])
        return (0, t, t)
    ev = ShardedEvaluator(measure, 8)
    golden = json.loads((GOLDEN / "ga_runs.json").read_text())
    run = next(r for r in golden if r["model"] == "separable" and r["seed"] == 1 and r["population"] == 12)
    res = ev.run_ga(seed=1)
    assert res["csv"] == run["csv"]
    c = ev.counters()
    assert {k: c[k] for k in run["counters"]} == run["counters"]
    assert c["elapsed_s"].hex() == run["elapsed_s"]
    with pytest.raises(Exception):
        ev.evaluate("101")
