"""Population-parallel fitness evaluation across ranks (one process per GPU, torch.distributed).

The reference evaluates a generation's batch with `jobs` independent workers in one process
(/root/reference/proj/src/evaluator.cpp:246-276).  Under the one-process-per-GPU launch contract the
same thing is done across ranks:

  * every rank runs the same deterministic GA (same seed, same outcomes => same populations);
  * `evaluate_all` dedupes the batch against the memo exactly like Evaluator::evaluate
    (evaluator.cpp:219-244: requests / distinct / cache_hits / backend_calls), assigns the unseen
    genomes to ranks, each rank measures only its share on its own GPU, and the outcomes are
    all-gathered as one small tensor (3 doubles per genome) -- that gather is the only
    communication; there is no collective on the data path;
  * assignment is longest-processing-time-first on a static cost estimate (a CPU-mapped matmul nest
    costs orders of magnitude more than anything else), so the expensive individuals are spread
    before the cheap ones fill in.

`measure` is any callable genome_str -> (status, time_s, wall_cost_s): `capi.Context.measure` on the
rank's GPU in production, a cost-model function in the CPU (gloo) tests.
"""
from __future__ import annotations

import ctypes as C
import time
from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import hostapi as H

Outcome = tuple  # (status, time_s, wall_cost_s)


class ShardedMeasureError(RuntimeError):
    """A rank's measure callable raised; raised on every rank of the group after the collective."""


def default_cost(genome: str) -> float:
    """Relative cost guess for the matrix application's genomes (only used to balance ranks)."""
    if len(genome) != 12:
        return 1.0
    nests = [(0, 2), (2, 2), (4, 2), (6, 2), (8, 3), (11, 1)]
    if any(genome[s:s + d].count("1") > 1 for s, d in nests):
        return 0.0                                   # infeasible: rejected without running
    cost = 1.0
    mm = genome[8:11]
    if mm == "000":
        cost += 1000.0                               # matmul nest on the CPU
    elif mm == "010":
        cost += 300.0                                # N GEMV launches, each reading all of bt
    elif mm == "001":
        cost += 3000.0                               # N^2 launches
    cost += 5.0 * sum(genome[s + 1] == "1" for s, d in nests[:4])   # N-launch inner loops
    cost += 2.0 * sum(genome[s:s + d] == "0" * d for s, d in nests[:4])  # cheap nests on the CPU
    return cost


def assign_lpt(genomes: Sequence[str], world: int, cost: Callable[[str], float] = default_cost) -> list[int]:
    """Owner rank per genome: longest-processing-time-first; ties broken by genome string so that every
    rank computes the same assignment."""
    order = sorted(range(len(genomes)), key=lambda i: (-cost(genomes[i]), genomes[i]))
    load = [0.0] * world
    owner = [0] * len(genomes)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += max(cost(genomes[i]), 1e-6)
    return owner


class ShardedEvaluator:
    """GenomeEvaluator semantics (evaluation.hpp:39-56) over the ranks of a process group."""

    def __init__(self, measure: Callable[[str], Outcome], gene_length: int, group=None,
                 device: torch.device | str = "cpu", cost: Callable[[str], float] = default_cost):
        self.measure, self.gene_length, self.group, self.cost = measure, gene_length, group, cost
        self.device = torch.device(device)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.memo: dict[str, Outcome] = {}
        self.requests = self.distinct = self.cache_hits = self.backend_calls = 0
        self.local_measurements = 0    # what THIS rank measured (tests pin the sharding with it)
        self._t0 = time.perf_counter()
        self.batch_wall: list[float] = []   # seconds since construction at the end of every evaluate_all call (run_ga: call g = generation g)

    def preload(self, genome: str, outcome: Outcome) -> None:
        """Seed the memo with an outcome obtained elsewhere, like the reference's Evaluator loading eval_cache.jsonl at
        construction (evaluator.cpp:150-176): later requests for the genome are cache hits on every rank and,
        as there, loading moves no counter.  Every rank must
        preload the same outcomes."""
        if len(genome) != self.gene_length:
            raise H.HostError(H.E_LENGTH, f"preload: genome length {len(genome)} does not match candidate count {self.gene_length}")
        self.memo[genome] = (int(outcome[0]), float(outcome[1]), float(outcome[2]))

    # -- GenomeEvaluator ---------------------------------------------------------------------------
    def evaluate(self, genome: str) -> Outcome:
        return self.evaluate_all([genome])[0]

    def evaluate_all(self, genomes: Sequence[str]) -> list[Outcome]:
        for g in genomes:
            if len(g) != self.gene_length:
                raise H.HostError(H.E_LENGTH, f"evaluate: genome length {len(g)} does not match candidate count {self.gene_length}")
        fresh: list[str] = []
        seen_in_batch = set()
        for g in genomes:
            self.requests += 1
            if g in self.memo or g in seen_in_batch:
                self.cache_hits += 1
            else:
                seen_in_batch.add(g)
                fresh.append(g)
                self.distinct += 1
                self.backend_calls += 1
        if fresh:
            owner = assign_lpt(fresh, self.world, self.cost)
            # columns: status, time_s, wall_cost_s, failed.  A rank whose measurement raises (MMX_E_CUDA, out of memory, ...)
            # still takes part in the collective and flags its row, so that no rank is left waiting in the all-reduce and a
            # failed row cannot be mistaken for a legitimate all-zero one (status 0 = Measured, time 0); the same error is
            # then raised on EVERY rank and nothing of the batch is memoised.
            mine = torch.zeros((len(fresh), 4), dtype=torch.float64)
            local_error: BaseException | None = None
            for i, g in enumerate(fresh):
                if owner[i] == self.rank:
                    try:
                        status, t, w = self.measure(g)
                    except Exception as e:  # noqa: BLE001 - reported on every rank below
                        local_error = local_error or e
                        mine[i, 3] = 1.0
                        continue
                    self.local_measurements += 1
                    mine[i, 0], mine[i, 1], mine[i, 2] = float(status), t, w
            if self.world > 1:
                # exactly one rank wrote each row, the others hold zeros: a SUM all-reduce is the gather
                buf = mine.to(self.device)
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
                mine = buf.cpu()
            failed = [fresh[i] for i in range(len(fresh)) if mine[i, 3].item() != 0.0]
            if failed:
                # roll the counters back: the batch did not happen (the reference memoises an exception per genome,
                # evaluator.cpp:206-211; across ranks the error object itself cannot travel, its existence does)
                self.requests -= len(genomes)
                self.cache_hits -= len(genomes) - len(fresh)
                self.distinct -= len(fresh)
                self.backend_calls -= len(fresh)
                msg = f"measurement failed on rank(s) owning {failed[:4]}{'...' if len(failed) > 4 else ''}"
                if local_error is not None:
                    raise ShardedMeasureError(f"{msg}: {local_error}") from local_error
                raise ShardedMeasureError(msg)
            for i, g in enumerate(fresh):
                self.memo[g] = (int(mine[i, 0].item()), float(mine[i, 1].item()), float(mine[i, 2].item()))
        self.batch_wall.append(time.perf_counter() - self._t0)
        return [self.memo[g] for g in genomes]

    def counters(self) -> dict:
        # elapsed_s in genome order, like Evaluator::counters (evaluator.cpp:285-290)
        elapsed = 0.0
        for g in sorted(self.memo):
            elapsed += self.memo[g][2]
        return {"requests": self.requests, "distinct": self.distinct, "cache_hits": self.cache_hits,
                "backend_calls": self.backend_calls, "elapsed_s": elapsed}

    # -- run_ga through the C++ host layer -----------------------------------------------------
    def run_ga(self, population=12, generations=12, crossover_rate=0.9, mutation_rate=0.05, seed=1, elite_count=1) -> dict:
        api = H.mine()
        batch_t = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint8), C.c_size_t, C.c_size_t, C.POINTER(H.Outcome), C.c_void_p)
        counters_t = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.c_void_p)
        failure: list[BaseException] = []

        def batch(bits, count, n, outs, _user):
            try:
                flat = np.ctypeslib.as_array(bits, shape=(count * n,))
                genomes = ["".join("1" if b else "0" for b in flat[i * n:(i + 1) * n]) for i in range(count)]
                for i, (status, t, w) in enumerate(self.evaluate_all(genomes)):
                    outs[i].status, outs[i].time_s, outs[i].wall_cost_s = status, t, w
                return 0
            except H.HostError as e:
                failure.append(e)
                return e.code
            except BaseException as e:  # noqa: BLE001 - must not unwind through C
                failure.append(e)
                return H.E_ERROR

        def counters(c4, elapsed, _user):
            c = self.counters()
            c4[0], c4[1], c4[2], c4[3] = c["requests"], c["distinct"], c["cache_hits"], c["backend_calls"]
            elapsed[0] = c["elapsed_s"]
            return 0

        params = H.GAParams(population, generations, crossover_rate, mutation_rate, seed, elite_count)
        csv = C.create_string_buffer(1 << 16)
        best = (C.c_uint8 * 64)()
        best_s, base_s = C.c_double(), C.c_double()
        bcb, ccb = batch_t(batch), counters_t(counters)
        rc = api.lib.mmxh_run_ga_external(C.c_size_t(self.gene_length), bcb, ccb, None, C.byref(params), csv,
                                          C.c_size_t(1 << 16), best, C.byref(best_s), C.byref(base_s))
        if rc < 0:
            if failure and not isinstance(failure[0], H.HostError):
                raise failure[0]
            api.check(rc)
        return {"csv": csv.value.decode(), "best_genome": "".join("1" if b else "0" for b in best[: self.gene_length]),
                "best_s": best_s.value, "baseline_s": base_s.value}
