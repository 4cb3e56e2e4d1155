"""The GA / sim-model restatement (paper_1806_01430_b200/host) against golden vectors produced by
the unmodified reference (tests/golden/generate_golden.py) and -- where oracle/_ref travels with
the snapshot -- against the reference itself, side by side.  Everything here is integer / RNG /
ordering work: the bar is bit-exact (byte-identical generations.csv)."""
import sys
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1806_01430_b200 import hostapi as H

sys.path.insert(0, str(Path(__file__).resolve().parent))
import refapi  # noqa: E402  (test-only loader of the compiled reference)

GOLDEN = Path(__file__).resolve().parent / "golden"
MODELS = GOLDEN / "models"
GENES = {"matrix12": 12, "separable": 8, "coupled": 10}


@pytest.fixture(scope="module")
def api():
    return H.mine()


@pytest.fixture(scope="module")
def ops():
    return json.loads((GOLDEN / "ga_operators.json").read_text())


def test_rng_draw_discipline(api, ops):
    for seed, entry in ops["rng"].items():
        seed = int(seed)
        assert api.rng_draws(seed, 3, 16) == entry["raw"]
        assert [int(x) for x in api.rng_draws(seed, 0, 16)] == entry["bit"]
        assert [x.hex() for x in api.rng_draws(seed, 1, 16)] == entry["real01"]
        assert [int(x) for x in api.rng_draws(seed, 2, 16, 11)] == entry["index11"]


def test_init_population_matches_reference(api, ops):
    for case in ops["init_population"]:
        assert api.init_population(case["a"], case["m"], case["seed"]) == case["genomes"]
    # the first individual of init_population(12, M=8, seed=1)
    assert api.init_population(12, 8, 1)[0] == "000001010001"


def test_fitness_known_answers(api, ops):
    # reference tests/test_ga.cpp:54-64
    assert api.fitness_from_time(4.0) == 0.5
    assert api.fitness_from_time(92.27) == 0.10410455682384989
    for case in ops["fitness_from_time"]:
        assert api.fitness_from_time(float.fromhex(case["t"])).hex() == case["fitness"]
    for t, rc in zip((0.0, -1.0, float("nan")), ops["fitness_nonpositive_rc"]):
        with pytest.raises(H.HostError) as e:
            api.fitness_from_time(t)
        assert e.value.code == rc == H.E_NONPOSITIVE


def test_assign_fitness_penalty(api, ops):
    for case in ops["assign_fitness"]:
        got = api.assign_fitness(case["status"], [float.fromhex(x) for x in case["time_s"]])
        assert [x.hex() for x in got] == case["fitness"]
    # failed individuals get 1e-3 x the smallest measured fitness; none measured -> 0
    assert api.assign_fitness([1, 2], [4.0, 0.0]) == [0.5, 0.5e-3]
    assert api.assign_fitness([2, 2], [0.0, 0.0]) == [0.0, 0.0]


def test_roulette_mutate_crossover_breed(api, ops):
    for case in ops["roulette"]:
        assert api.roulette([float.fromhex(x) for x in case["fitness"]], case["count"], case["seed"]) == case["picks"]
    with pytest.raises(H.HostError) as e:
        api.roulette([0.0, 0.0], 1, 1)
    assert e.value.code == ops["roulette_zero_total_rc"] == H.E_ZERO_FITNESS
    for case in ops["mutate"]:
        assert api.mutate(case["genome"], case["pm"], case["seed"]) == case["out"]
    for case in ops["one_point_crossover"]:
        assert list(api.one_point_crossover(case["p1"], case["p2"], case["seed"])) == [case["c1"], case["c2"]]
    for case in ops["breed"]:
        got = api.breed(case["genomes"], [float.fromhex(x) for x in case["fitness"]], case["pc"], case["pm"], case["elite"],
                        case["seed"], case["skip"])
        assert got == case["next"], case


@pytest.mark.parametrize("name", sorted(GENES))
def test_model_time_of_every_genome(api, name):
    want = np.load(GOLDEN / f"model_times_{name}.npy")
    got = api.model_time_all(MODELS / f"{name}.json", GENES[name])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    best = json.loads((GOLDEN / f"model_best_{name}.json").read_text())
    g, t = api.exhaustive_best(MODELS / f"{name}.json", GENES[name])
    assert (g, t.hex()) == (best["genome"], best["time_s"])


def test_model_known_optima(api):
    # reference tests/test_sim_model.cpp:60-82
    assert api.exhaustive_best(MODELS / "matrix12.json", 12) == ("100000000000", pytest.approx(0.00243, abs=1e-12))
    assert api.exhaustive_best(MODELS / "separable.json", 8)[0] == "11101001"
    assert api.exhaustive_best(MODELS / "coupled.json", 10)[0] == "1111100000"


def golden_runs():
    return json.loads((GOLDEN / "ga_runs.json").read_text())


@pytest.mark.parametrize("idx", range(len(golden_runs())))
def test_run_ga_is_byte_identical_to_the_reference(api, idx):
    run = golden_runs()[idx]
    with H.Evaluator.from_sim(api, MODELS / f"{run['model']}.json") as ev:
        got = ev.run_ga(run["population"], run["generations"], run["crossover_rate"], run["mutation_rate"], run["seed"],
                        run["elite_count"], genes=GENES[run["model"]])
        assert got["csv"] == run["csv"]
        assert got["best_genome"] == run["best_genome"]
        assert got["best_s"].hex() == run["best_s"] and got["baseline_s"].hex() == run["baseline_s"]
        c = ev.counters()
        assert {k: c[k] for k in run["counters"]} == run["counters"]
        assert c["elapsed_s"].hex() == run["elapsed_s"]


def test_survey_appendix_b_rows(api):
    runs = golden_runs()
    assert "12,0.00255,36.1843137,101000011000,18.1448781,77,57" in runs[0]["csv"]
    assert runs[1]["csv"].splitlines()[-1] == "40,0.00243,37.9711934,100000000000,18.7890421,1215,1307"


def test_jobs_do_not_change_the_trajectory(api):
    run = golden_runs()[0]
    with H.Evaluator.from_sim(api, MODELS / "matrix12.json", jobs=6) as ev:
        assert ev.run_ga()["csv"] == run["csv"]


def test_rerun_from_cache_file_touches_no_backend(api, tmp_path):
    # reference tests/test_cli.cpp:371-394 / test_evaluator.cpp:202-241
    cache = tmp_path / "cache" / "eval_cache.jsonl"
    run = golden_runs()[0]
    with H.Evaluator.from_sim(api, MODELS / "matrix12.json", cache_file=cache) as ev:
        first = ev.run_ga()
        cold = ev.counters()
    lines = cache.read_text().splitlines()
    assert len(lines) == cold["distinct"] == 77
    # byte-compatible with the file the reference writes (key order, number formatting)
    assert lines[:16] == (GOLDEN / "eval_cache_sample.jsonl").read_text().splitlines()
    with H.Evaluator.from_sim(api, MODELS / "matrix12.json", cache_file=cache) as ev:
        second = ev.run_ga()
        warm = ev.counters()
    assert second["csv"] == first["csv"] == run["csv"]
    assert warm["backend_calls"] == 0 and warm["distinct"] == cold["distinct"]
    assert warm["elapsed_s"] == cold["elapsed_s"]
    assert len(cache.read_text().splitlines()) == 77   # nothing appended


def test_ga_failure_modes(api):
    # reference tests/test_ga.cpp:435-484
    def all_fail(g):
        return (1, 0.0, 0.0) if "1" in g else (0, 1.0, 0.1)   # only the baseline measures
    with H.Evaluator.from_callback(api, 6, all_fail) as ev:
        with pytest.raises(H.HostError) as e:
            ev.run_ga(population=4, generations=3, genes=6)
        assert e.value.code in (H.E_ZERO_FITNESS,)   # every individual failed -> empty wheel
    with H.Evaluator.from_callback(api, 6, lambda g: (2, 0.0, 0.0)) as ev:
        with pytest.raises(H.HostError) as e:
            ev.run_ga(population=4, generations=3, genes=6)
        assert e.value.code == H.E_UNAVAILABLE       # baseline not measurable
    with H.Evaluator.from_callback(api, 6, lambda g: (0, 1.0, 0.1)) as ev:
        for bad in (dict(population=1), dict(generations=0), dict(crossover_rate=1.5), dict(mutation_rate=-0.1),
                    dict(elite_count=0), dict(population=4, elite_count=4)):
            with pytest.raises(H.HostError) as e:
                ev.run_ga(genes=6, **bad)
            assert e.value.code == H.E_CONFIG


def test_timeouts_score_as_measured_and_failures_are_penalised(api):
    # Timeout -> Measured with time = budget (ga.cpp:206-211); CompileError -> Failed
    def fn(g):
        k = g.count("1")
        if k == 0:
            return (0, 10.0, 0.1)
        if g[0] == "1":
            return (3, 30.0, 30.0)       # timeout: budget 30 s
        if g[1] == "1":
            return (1, 0.0, 0.01)        # compile error
        return (0, 10.0 - k, 0.1)
    with H.Evaluator.from_callback(api, 5, fn) as ev:
        res = ev.run_ga(population=8, generations=6, seed=3, genes=5)
    rows = res["csv"].splitlines()
    assert rows[2].split(",")[0] == "1" and float(rows[-1].split(",")[1]) <= 10.0
    assert res["best_genome"][0] == "0"   # a timed-out genome never wins against measured ones


REF = refapi.reference()


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built (needs /root/reference)")
def test_side_by_side_with_the_reference_on_random_operator_inputs(api):
    rs = np.random.RandomState(42)
    for trial in range(40):
        a, m = int(rs.randint(2, 14)), int(rs.randint(2, 12))
        seed, skip = int(rs.randint(1, 10 ** 6)), int(rs.randint(0, 50))
        genomes = ["".join(str(x) for x in rs.randint(0, 2, a)) for _ in range(m)]
        fitness = [float(x) for x in rs.rand(m)]
        if trial % 5 == 0:
            fitness = [round(x, 1) for x in fitness]   # provoke ties
        pc, pm, elite = float(rs.rand()), float(rs.rand() * 0.5), int(rs.randint(1, m))
        assert api.breed(genomes, fitness, pc, pm, elite, seed, skip) == REF.breed(genomes, fitness, pc, pm, elite, seed, skip)
        assert api.init_population(a, m, seed) == REF.init_population(a, m, seed)
        assert api.roulette(fitness, 20, seed) == REF.roulette(fitness, 20, seed)
        assert api.mutate(genomes[0], pm, seed) == REF.mutate(genomes[0], pm, seed)
        assert api.one_point_crossover(genomes[0], genomes[1], seed) == REF.one_point_crossover(genomes[0], genomes[1], seed)
        status = [int(x) for x in rs.randint(1, 3, m)]
        times = [float(x) + 0.01 for x in rs.rand(m)]
        assert api.assign_fitness(status, times) == REF.assign_fitness(status, times)
