"""The Evaluator contract, transcribed from the reference's tests/test_evaluator.cpp:103-262 and
run against this repo's mmxhost::Evaluator through a scripted callback backend -- and, where
oracle/_ref is present, run identically against the reference's own Evaluator."""
import sys
from pathlib import Path
import threading
import time

import pytest

from paper_1806_01430_b200 import hostapi as H

sys.path.insert(0, str(Path(__file__).resolve().parent))
import refapi  # noqa: E402  (test-only loader of the compiled reference)

APIS = [pytest.param(H.mine(), id="mmxhost")]
if refapi.reference() is not None:
    APIS.append(pytest.param(refapi.reference(), id="reference"))

MEASURED, COMPILE_ERROR, RUNTIME_ERROR, TIMEOUT = range(4)


class Script:
    """ScriptBackend (tests/test_util.hpp:55-81): counts calls and the maximum in flight."""

    def __init__(self, fn):
        self.fn, self.calls, self.in_flight, self.max_in_flight = fn, 0, 0, 0
        self.lock = threading.Lock()

    def __call__(self, genome):
        with self.lock:
            self.calls += 1
            self.in_flight += 1
            self.max_in_flight = max(self.max_in_flight, self.in_flight)
        try:
            return self.fn(genome)
        finally:
            with self.lock:
                self.in_flight -= 1


@pytest.mark.parametrize("api", APIS)
def test_repeat_evaluations_hit_the_memo(api):           # test_evaluator.cpp:103-123
    script = Script(lambda g: (MEASURED, 2.5, 0.3))
    with H.Evaluator.from_callback(api, 4, script) as ev:
        first = ev.evaluate("1010")
        for _ in range(5):
            assert ev.evaluate("1010") == first
        assert script.calls == 1
        c = ev.counters()
        assert (c["requests"], c["distinct"], c["cache_hits"], c["backend_calls"], c["elapsed_s"]) == (6, 1, 5, 1, 0.3)


@pytest.mark.parametrize("api", APIS)
def test_evaluate_all_deduplicates_and_aligns(api):      # :125-148
    script = Script(lambda g: (MEASURED, 1.0 + g.count("1"), 0.1))
    with H.Evaluator.from_callback(api, 3, script, jobs=4) as ev:
        ev.evaluate("100")
        assert script.calls == 1
        batch = ["110", "100", "110", "111", "100"]
        outs = ev.evaluate_all(batch)
        assert [o[1] for o in outs] == [1.0 + g.count("1") for g in batch]
        assert script.calls == 3
        c = ev.counters()
        assert (c["requests"], c["distinct"], c["cache_hits"]) == (6, 3, 3)


@pytest.mark.parametrize("api", APIS)
def test_concurrent_duplicates_reach_the_backend_once(api):   # :150-164
    def slow(g):
        time.sleep(0.03)
        return (MEASURED, 1.5, 0.2)
    script = Script(slow)
    with H.Evaluator.from_callback(api, 4, script, jobs=4) as ev:
        outs = ev.evaluate_all(["0110"] * 8)
        assert all(o[1] == 1.5 for o in outs)
        assert script.calls == 1
        c = ev.counters()
        assert (c["requests"], c["distinct"], c["cache_hits"]) == (8, 1, 7)


@pytest.mark.parametrize("api", APIS)
def test_at_most_jobs_measurements_at_once(api):         # :166-182
    def slow(g):
        time.sleep(0.03)
        return (MEASURED, 1.0 + g.count("1"), 0.1)
    script = Script(slow)
    with H.Evaluator.from_callback(api, 4, script, jobs=4) as ev:
        batch = ["".join(str((i >> k) & 1) for k in range(4)) for i in range(8)]
        ev.evaluate_all(batch)
        assert script.calls == 8
        assert 2 <= script.max_in_flight <= 4


@pytest.mark.parametrize("api", APIS)
def test_backend_exceptions_are_remembered_per_genome(api):   # :184-194
    def fn(g):
        if g[0] == "1":
            raise H.ToolchainMissingSignal()
        return (MEASURED, 1.0, 0.1)
    script = Script(fn)
    with H.Evaluator.from_callback(api, 2, script) as ev:
        for _ in range(2):
            with pytest.raises(H.HostError) as e:
                ev.evaluate("10")
            assert e.value.code == H.E_TOOLCHAIN
        assert script.calls == 1
        assert ev.evaluate("01")[0] == MEASURED
        # a failing genome inside a batch: first exception rethrown after the batch drained
        with pytest.raises(H.HostError):
            ev.evaluate_all(["01", "10", "00"])


@pytest.mark.parametrize("api", APIS)
def test_wrong_genome_length_is_rejected(api):           # :196-200
    with H.Evaluator.from_callback(api, 8, lambda g: (MEASURED, 1.0, 0.1)) as ev:
        with pytest.raises(H.HostError) as e:
            ev.evaluate("1010")
        assert e.value.code == H.E_LENGTH


@pytest.mark.parametrize("api", APIS)
def test_disk_cache_makes_reruns_free(api, tmp_path):    # :202-241
    cache = tmp_path / "cache" / "evals.jsonl"
    genomes = ["00000000", "11101001", "10000000"]
    fn = lambda g: (MEASURED, 0.5 + 0.125 * g.count("1"), 0.25 + 0.125 * g.count("1"))  # noqa: E731
    with H.Evaluator.from_callback(api, 8, fn, cache_file=cache) as ev:
        first = [ev.evaluate(g) for g in genomes]
        ev.evaluate(genomes[0])
        cold = ev.counters()
    assert (cold["requests"], cold["distinct"], cold["cache_hits"], cold["backend_calls"]) == (4, 3, 1, 3)
    assert len(cache.read_text().splitlines()) == 3
    script = Script(fn)
    with H.Evaluator.from_callback(api, 8, script, cache_file=cache) as ev:
        assert [ev.evaluate(g) for g in genomes] == first
        c = ev.counters()
        assert (c["requests"], c["distinct"], c["cache_hits"], c["backend_calls"]) == (3, 3, 0, 0)
        assert c["elapsed_s"] == cold["elapsed_s"]
    assert script.calls == 0


@pytest.mark.parametrize("api", APIS)
def test_bad_cache_lines_are_skipped(api, tmp_path):     # :243-262
    cache = tmp_path / "evals.jsonl"
    cache.write_text("\n".join([
        "not json at all",
        '{"genome":"10","status":"measured","time_s":1.5,"wall_cost_s":0.2}',
        '{"genome":"1x","status":"measured","time_s":1.0,"wall_cost_s":0.1}',       # not a bit string
        '{"genome":"101","status":"measured","time_s":1.0,"wall_cost_s":0.1}',      # wrong length
        '{"genome":"01","status":"exploded","time_s":1.0,"wall_cost_s":0.1}',       # unknown status
        '{"genome":"11","status":"measured","time_s":0.0,"wall_cost_s":0.1}',       # measured but t <= 0
        '{"genome":"00","status":"timeout","time_s":30.0,"wall_cost_s":30.5}',
        '[1,2,3]',
        "",
    ]) + "\n")
    script = Script(lambda g: (MEASURED, 9.0, 0.9))
    with H.Evaluator.from_callback(api, 2, script, cache_file=cache) as ev:
        assert ev.evaluate("10") == (MEASURED, 1.5, 0.2)
        assert ev.evaluate("00") == (TIMEOUT, 30.0, 30.5)
        assert script.calls == 0
        for g in ("01", "11"):
            assert ev.evaluate(g) == (MEASURED, 9.0, 0.9)
        assert script.calls == 2


@pytest.mark.parametrize("api", APIS)
def test_outcome_status_passthrough_and_names(api):
    table = {"0001": (COMPILE_ERROR, 0.0, 0.01), "0010": (RUNTIME_ERROR, 0.0, 0.02), "0100": (TIMEOUT, 10.0, 10.1)}
    with H.Evaluator.from_callback(api, 4, lambda g: table.get(g, (MEASURED, 1.0, 0.1))) as ev:
        for g, want in table.items():
            assert ev.evaluate(g) == want
    assert [api.status_name(s) for s in range(4)] == ["measured", "compile_error", "runtime_error", "timeout"]


def test_cache_number_formatting_matches_nlohmann():
    # what the reference's ordered_json::dump() prints for these doubles (layout rules of nlohmann's
    # format_buffer: plain decimal for decimal exponents in (-4, 15], else d.ddde+XX).  Digits come from
    # std::to_chars (shortest round trip); nlohmann's Grisu2 is one digit longer for ~0.35% of random
    # doubles -- both spellings parse back to the same double.
    cases = {0.09227000000000007: "0.09227000000000007", 1.0: "1.0", 0.0: "0.0", 120.0: "120.0", 1e-5: "1e-05",
             0.0001: "0.0001", 0.00243: "0.00243", 1e14: "100000000000000.0", 1e15: "1e+15", 123456.789: "123456.789",
             5.5e-3: "0.0055", 2.5e-7: "2.5e-07", -0.5: "-0.5"}
    for v, want in cases.items():
        assert H.dump_number(v) == want


# ---- longest-first scheduling of a batch (mmxhost only: the reference pulls in input order, evaluator.cpp:254-273) ----

def test_cost_hint_starts_the_longest_genome_first():
    api = H.mine()
    started, lock = [], threading.Lock()

    def record(g):
        with lock:
            started.append(g)
        time.sleep(0.05)        # long enough that every worker has pulled its first genome before any pulls a second
        return (MEASURED, 1.0 + g.count("1"), 0.1)
    batch = ["0001", "0011", "0111", "1111", "0000"]
    with H.Evaluator.from_callback(api, 4, record, jobs=1) as ev:
        ev.set_costs(batch, [g.count("1") for g in batch])
        # jobs == 1 evaluates in input order (the serial path is the reference's); the hint only orders the worker pull
        ev.evaluate_all(batch)
        assert started == batch
    started.clear()
    with H.Evaluator.from_callback(api, 4, record, jobs=2) as ev:
        ev.set_costs(batch, [g.count("1") for g in batch])
        outs = ev.evaluate_all(batch)
        assert [o[1] for o in outs] == [1.0 + g.count("1") for g in batch]      # outcomes stay aligned with the input
        assert set(started[:2]) == {"1111", "0111"}                             # the two dearest start first
        assert started[-1] == "0000"


def test_cost_hint_shortens_a_batch_with_one_slow_genome():
    api = H.mine()

    def run(hint):
        def timed(g):
            time.sleep(0.30 if g == "1111" else 0.05)
            return (MEASURED, 1.0, 0.0)
        batch = ["0001", "0010", "0100", "1000", "0011", "0110", "1111"]       # the slow one is last in input order
        with H.Evaluator.from_callback(api, 4, timed, jobs=2) as ev:
            if hint:
                ev.set_costs(batch, [0.30 if g == "1111" else 0.05 for g in batch])
            t0 = time.perf_counter()
            ev.evaluate_all(batch)
            return time.perf_counter() - t0
    unhinted, hinted = run(False), run(True)
    assert unhinted > 0.42          # 3 rounds of 0.05 on two workers, then 0.30 alone
    assert hinted < 0.38            # 0.30 on one worker while the other takes the six short ones


def test_predicted_cost_ranks_host_contraction_and_launch_trains_over_offload():
    n = 1024
    all_offloaded, cpu_matmul, cpu_small_nest, all_cpu = "101010101001", "101010100001", "101010001001", "0" * 12
    k_train = "101010100011"                                                    # gene 10: one launch per (i, j)
    c = {g: H.predicted_cost(g, n=n) for g in (all_offloaded, cpu_matmul, cpu_small_nest, all_cpu, k_train)}
    assert c[all_offloaded] < c[cpu_small_nest] < c[cpu_matmul] <= c[all_cpu]
    assert c[k_train] > 1000 * c[all_offloaded]                                 # N^2 launches dominate
    assert H.predicted_cost("110000000000", n=n) == 0.0                         # infeasible: produced on the spot
    assert H.predicted_cost(all_cpu, n=n, host_threads=8) < c[all_cpu]
    assert H.predicted_cost(all_cpu, n=n, repetitions=3, warmup=1) == pytest.approx(4 * c[all_cpu])
    assert H.predicted_cost(all_cpu, n=8192, timeout_s=1.0) == 1.0              # capped at the timeout
