"""Cost-model calibration: measured genome times -> plan model -> the reference's model file.

CPU tests use synthetic "measurements" generated from a known plan model (through this repo's planner, mmx_plan), so the
fit, the projection onto the reference's additive form and the file format can be checked exactly; the file is parsed by
this repo's parse_model and, where oracle/_ref is built, by the reference's (sim_model.cpp:157-236).  The GPU run of the
same pipeline is tools/calibrate.py.
"""
import sys
from pathlib import Path
import numpy as np
import pytest

from paper_1806_01430_b200 import hostapi as H

sys.path.insert(0, str(Path(__file__).resolve().parent))
import refapi  # noqa: E402  (test-only loader of the compiled reference)

N = 256
# serial, cpu[6], loop[12], h2d s/B, d2h s/B, per-transfer s -- the shape of a B200 at the fixture size
TRUTH = np.array([5e-6, 40e-6, 40e-6, 30e-6, 120e-6, 8.3e-3, 1e-6,
                  3e-6, 400e-6, 3e-6, 400e-6, 3e-6, 380e-6, 4e-6, 450e-6, 10e-6, 1.1e-3, 0.11, 5e-6,
                  1 / 25e9, 1 / 22e9, 8e-6])


def genome_of(mask):
    return "".join("1" if (mask >> k) & 1 else "0" for k in range(12))


@pytest.fixture(scope="module")
def truth_times():
    t = H.plan_model_times(TRUTH, N)
    assert (t > 0).sum() == 648          # the feasible genomes of the application
    return t


def samples(times, noise=0.0, seed=0):
    rs = np.random.RandomState(seed)
    masks = [m for m in range(4096) if times[m] > 0]
    return [genome_of(m) for m in masks], [times[m] * (1.0 + noise * rs.uniform(-1, 1)) for m in masks]


def test_fit_reproduces_noise_free_measurements(truth_times):
    genomes, times = samples(truth_times)
    cal = H.calibrate(genomes, times, N)
    assert cal["report"]["samples"] == 648
    assert cal["report"]["fit_max_rel_err"] < 1e-6
    refit = H.plan_model_times(cal["plan"], N)
    ok = truth_times > 0
    assert np.allclose(refit[ok], truth_times[ok], rtol=1e-6, atol=0)
    assert (refit[~ok] == -1).all()
    best = int(np.argmin(np.where(ok, truth_times, np.inf)))
    assert cal["plan_best"] == genome_of(best) and cal["plan_best"].startswith("1010101010")   # every matrix nest offloaded at its outer loop


def test_fit_tolerates_measurement_noise(truth_times):
    genomes, times = samples(truth_times, noise=0.02, seed=7)
    cal = H.calibrate(genomes, times, N)
    assert cal["report"]["fit_rms_rel_err"] < 0.03 and cal["report"]["fit_max_rel_err"] < 0.12
    assert cal["plan_best"].startswith("1010101010")


def test_too_few_samples_is_a_model_error(truth_times):
    genomes, times = samples(truth_times)
    with pytest.raises(H.HostError) as e:
        H.calibrate(genomes[:10], times[:10], N)
    assert e.value.code == -10     # ModelError


def test_projection_onto_the_reference_cost_model(truth_times, tmp_path):
    genomes, times = samples(truth_times)
    cal = H.calibrate(genomes, times, N)
    path = tmp_path / "calibrated.json"
    path.write_text(cal["model_json"])
    mine = H.mine().model_time_all(path, 12)                       # parse_model + model_time, this repo
    plan = H.plan_model_times(cal["plan"], N)
    feasible = plan > 0
    # infeasible genomes are exactly the model's fail set (-1 from model_time_all)
    assert ((mine < 0) == ~feasible).all()
    # offload depths of one nest that are BOTH faster than the CPU cannot be represented additively: here the GEMV
    # form of the matmul nest (gene 9); everything not using it is exact
    assert cal["report"]["inexact_loops"] == 1
    uses9 = np.array([(m >> 9) & 1 == 1 for m in range(4096)])
    exact = feasible & ~uses9
    assert np.allclose(mine[exact], plan[exact], rtol=1e-9, atol=1e-15)
    assert (mine[feasible & uses9] >= plan[feasible & uses9] * (1 - 1e-9)).all()   # the residual only ever over-estimates
    # both models agree on the optimum, and exhaustive_best over the file finds it
    assert cal["cost_best"] == cal["plan_best"]
    best, t = H.mine().exhaustive_best(path, 12)
    assert best == cal["cost_best"] and t == pytest.approx(cal["report"]["cost_best_s"], rel=1e-12)
    ref = refapi.reference()
    if ref is not None:                                            # the reference parses the same file to the same times
        theirs = ref.model_time_all(path, 12)
        assert np.array_equal(theirs < 0, mine < 0)
        assert np.array_equal(theirs[feasible].view(np.uint64), mine[feasible].view(np.uint64))
        assert ref.exhaustive_best(path, 12)[0] == best


def test_ga_on_the_calibrated_model_finds_the_exhaustive_optimum(truth_times, tmp_path):
    genomes, times = samples(truth_times)
    cal = H.calibrate(genomes, times, N)
    path = tmp_path / "calibrated.json"
    path.write_text(cal["model_json"])
    with H.Evaluator.from_sim(H.mine(), path) as ev:
        res = ev.run_ga(population=64, generations=40, seed=1)
    assert res["best_genome"] == cal["cost_best"]
