"""The callers of the hot path: loop-catalogue scan, variant rendering, config loading and
the `tune` / `report` commands of the C++ host layer, against golden outputs of the UNMODIFIED reference
(tests/golden/scan_cases.json, tests/golden/tune_sim/runs.json, made by tests/golden/generate_golden.py from
scan_loops / render_variant / cmd_tune / cmd_report) -- byte for byte.  Runs without a GPU."""
import json
import subprocess
from pathlib import Path

import pytest

from paper_1806_01430_b200 import capi, hostapi as H

GOLDEN = Path(__file__).resolve().parent / "golden"
BIN = Path(capi.LIB_DIR).parent / "bin" / "mmx_tune"


@pytest.fixture(scope="module")
def api():
    return H.mine()


@pytest.fixture(scope="module")
def matmul_source(api):
    """fixtures/matmul.c, recovered from the reference's own rendering of it (render then strip is the identity)."""
    return H.strip_directives(api, (GOLDEN / "rendered_best.c").read_text())


def fnv(text: str) -> str:
    h = 0xcbf29ce484222325
    for b in text.encode():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


# ---- scan_loops / render_variant -------------------------------------------------------------------------

def test_scanner_matches_the_reference_on_tricky_sources(api):
    cases = json.loads((GOLDEN / "scan_cases.json").read_text())
    assert len(cases) >= 6
    for name, case in cases.items():
        rows = [[r[k] for k in ("id", "line", "depth", "header_start", "body_begin", "body_end", "indent_len")]
                for r in H.scan_loops(api, case["text"], name)]
        assert rows == case["rows"], name
        for genome, rendered in case["renders"].items():
            assert H.render_variant(api, case["text"], genome) == rendered, (name, genome)
            assert H.strip_directives(api, rendered) == case["text"]


def test_catalogue_of_the_matrix_application(api, matmul_source):
    """The scanned catalogue equals the reference's (catalogue.json) and the one the kernel library serves."""
    golden = json.loads((GOLDEN / "catalogue.json").read_text())
    mine = H.scan_loops(api, matmul_source, "matmul.c")
    assert [(r["id"], r["line"], r["depth"]) for r in mine] == [(g["id"], g["line"], g["depth"]) for g in golden]
    assert [(r["gene"], r["line"], r["depth"]) for r in capi.loop_catalogue()] == [(g["id"], g["line"], g["depth"]) for g in golden]


def test_render_matches_the_reference(api, matmul_source):
    assert H.render_variant(api, matmul_source, "100000000000") == (GOLDEN / "rendered_best.c").read_text()
    assert H.render_variant(api, matmul_source, "101010101001") == (GOLDEN / "rendered_all_nests.c").read_text()
    assert H.render_variant(api, matmul_source, "0" * 12) == matmul_source
    with pytest.raises(H.HostError) as e:
        H.render_variant(api, matmul_source, "101")
    assert e.value.code == H.E_LENGTH


def test_unterminated_input_is_a_scan_error(api):
    for bad in ("void f(void) { for (;;) { }", "/* never closed\nint x;", "char* s = \"open;\n"):
        with pytest.raises(H.HostError):
            H.scan_loops(api, bad)


# ---- tune / report -----------------------------------------------------------------------------------------

def _workspace(tmp_path, matmul_source, cfg):
    (tmp_path / "matmul.c").write_text(matmul_source)
    (tmp_path / "model.json").write_bytes((GOLDEN / "models" / "matrix12.json").read_bytes())
    (tmp_path / "cfg.json").write_text(json.dumps(cfg))
    return tmp_path / "cfg.json"


@pytest.mark.parametrize("run", ["default_seed1", "m8_t6_seed7", "m64_t40_seed1"])
def test_tune_artifacts_are_byte_identical_to_the_reference(api, matmul_source, tmp_path, run):
    golden = json.loads((GOLDEN / "tune_sim" / "runs.json").read_text())[run]
    cfg_path = _workspace(tmp_path, matmul_source, golden["config"])
    rc, out, err = H.cmd_tune(api, cfg_path)
    assert rc == 0, err
    norm = lambda s: s.replace(str(tmp_path), "@TMP@")  # noqa: E731
    assert norm(out) == golden["stdout"]
    work = tmp_path / "work"
    for rel, text in golden["files"].items():
        assert norm((work / rel).read_text()) == text, rel
    best = (work / "best" / "matmul.c").read_text()
    assert fnv(best) == golden["best_genome_render_sha"]
    assert best == H.render_variant(api, matmul_source, golden["best_is_render_of"])
    rc, rout, rerr = H.cmd_report(api, work)
    assert rc == 0 and rout == golden["report_stdout"], rerr
    # a rerun replays from eval_cache.jsonl: same artifacts, zero backend calls (test_cli.cpp:371-394)
    rc, out2, _ = H.cmd_tune(api, cfg_path)
    assert rc == 0 and ", 0 backend calls" in out2
    assert norm((work / "generations.csv").read_text()) != "" and (work / "summary.json").read_text() == golden["files"]["summary.json"]


def test_seed_and_sim_overrides(api, matmul_source, tmp_path):
    cfg_path = _workspace(tmp_path, matmul_source, {"source": "matmul.c", "workdir": "work", "ga": {"seed": 5},
                                                     "cuda": {"n": 64}})
    # --sim replaces the configured backend, --seed the configured seed: the run equals the golden seed-1 run
    rc, out, err = H.cmd_tune(api, cfg_path, seed=1, sim_model=tmp_path / "model.json")
    assert rc == 0, err
    golden = json.loads((GOLDEN / "tune_sim" / "runs.json").read_text())["default_seed1"]
    assert (tmp_path / "work" / "generations.csv").read_text() == golden["files"]["generations.csv"]
    resolved = json.loads((tmp_path / "work" / "config.resolved.json").read_text())
    assert resolved["ga"]["seed"] == 1 and "cuda" not in resolved and resolved["sim_model"].endswith("model.json")


def test_the_command_line_binary(matmul_source, tmp_path):
    golden = json.loads((GOLDEN / "tune_sim" / "runs.json").read_text())["m8_t6_seed7"]
    cfg_path = _workspace(tmp_path, matmul_source, golden["config"])
    p = subprocess.run([str(BIN), "tune", str(cfg_path)], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0, p.stderr
    assert p.stdout.replace(str(tmp_path), "@TMP@") == golden["stdout"]
    assert (tmp_path / "work" / "generations.csv").read_text() == golden["files"]["generations.csv"]
    p = subprocess.run([str(BIN), "report", str(tmp_path / "work")], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and p.stdout == golden["report_stdout"]
    p = subprocess.run([str(BIN), "analyze", str(cfg_path)], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and "loops: 12" in p.stdout and "gene length: 12" in p.stdout
    assert subprocess.run([str(BIN), "tune"], capture_output=True).returncode == 2


BASE = {"source": "matmul.c", "workdir": "work", "sim_model": "model.json"}


@pytest.mark.parametrize("cfg,code,needle", [
    ({**BASE, "sorce": "x"}, 2, "unknown key 'sorce'"),
    ({"workdir": "work", "sim_model": "model.json"}, 2, "needs a 'source' entry"),
    ({**BASE, "cuda": {"n": 256}}, 2, "exactly one of"),
    ({"source": "matmul.c", "workdir": "work"}, 2, "exactly one of"),
    ({"source": "matmul.c", "workdir": "work", "toolchain": {"compile_cmd": "nvc", "bench_cmd": "x"}}, 2, "not part of this build"),
    ({**BASE, "ga": {"population": 1}}, 2, ""),
    ({**BASE, "ga": {"seed": -1}}, 2, "non-negative"),
    ({**BASE, "jobs": 0}, 2, "'jobs' must be at least 1"),
    ({**BASE, "candidates": "some"}, 2, "'candidates' must be"),
    ({**BASE, "source": "missing.c"}, 2, "cannot read source file"),
    ({**BASE, "sim_model": "nope.json"}, 2, ""),
    ({**BASE, "candidates": "outermost"}, 2, "sim model has 12 loops but the source has 6 candidates"),
    ({"source": "matmul.c", "workdir": "work", "cuda": {"n": 64, "dtype": "f16"}}, 2, "'dtype' must be"),
    ({"source": "matmul.c", "workdir": "work", "cuda": {"n": 64, "devices": []}}, 2, "'devices'"),
    ({"source": "matmul.c", "workdir": "work", "cuda": {"n": 64, "threads": 2}}, 2, "unknown key 'threads' in 'cuda'"),
])
def test_config_errors_map_to_exit_codes(api, matmul_source, tmp_path, cfg, code, needle):
    cfg_path = _workspace(tmp_path, matmul_source, cfg)
    rc, out, err = H.cmd_tune(api, cfg_path)
    assert rc == code, (rc, err)
    assert err.startswith("tune: ") and needle in err


def test_cuda_backend_needs_the_matrix_application_and_a_device(api, matmul_source, tmp_path):
    import torch
    other = tmp_path / "other"
    other.mkdir()
    cfg_path = _workspace(other, "void f(int n, double* a) {\n  for (int i = 0; i < n; ++i) a[i] = 0.0;\n}\n",
                          {"source": "matmul.c", "workdir": "work", "cuda": {"n": 64}})
    rc, _, err = H.cmd_tune(api, cfg_path)
    assert rc == 2 and "has no kernel for loop 0" in err and "matches no kernel idiom" in err
    # loops the library does have kernels for, but not the application the executor is wired to
    third = tmp_path / "third"
    third.mkdir()
    cfg_path = _workspace(third, "double c[8][8];\nvoid z(void) {\n  for (int i = 0; i < 8; i++)\n    for (int j = 0; j < 8; j++)\n      c[i][j] = 0.0;\n}\n",
                          {"source": "matmul.c", "workdir": "work", "cuda": {"n": 64}})
    rc, _, err = H.cmd_tune(api, cfg_path)
    assert rc == 2 and "loop catalogue of the matrix application" in err
    rc, out, _ = H.cmd_analyze(api, cfg_path)           # analyze needs no device: static probe + kernel matcher
    assert rc == 0 and "loop 0: line 3, depth 0 -> candidate [kernel: fill2d<zero>]" in out and "[kernel: fill_row<zero>]" in out
    if not torch.cuda.is_available():
        # no CPU fallback: the measuring tool is absent -> ToolchainMissing -> exit 4 (commands.cpp:172)
        cfg_path = _workspace(tmp_path, matmul_source, {"source": "matmul.c", "workdir": "work", "cuda": {"n": 64}})
        rc, _, err = H.cmd_tune(api, cfg_path)
        assert rc == 4, err


def test_report_rejects_corrupted_logs(api, matmul_source, tmp_path):
    golden = json.loads((GOLDEN / "tune_sim" / "runs.json").read_text())["m8_t6_seed7"]
    cfg_path = _workspace(tmp_path, matmul_source, golden["config"])
    assert H.cmd_tune(api, cfg_path)[0] == 0
    work = tmp_path / "work"
    assert H.cmd_report(api, tmp_path / "nowhere")[0] == 2          # MissingLog
    csv = (work / "generations.csv").read_text().splitlines()
    rows = csv[:2] + [csv[2].replace(csv[2].split(",")[1], "9.0", 1)] + csv[3:]
    (work / "generations.csv").write_text("\n".join(rows) + "\n")
    rc, _, err = H.cmd_report(api, work)
    assert rc == 1 and "best time regresses" in err
    (work / "generations.csv").write_text("generation,best\n")
    assert H.cmd_report(api, work)[0] == 1


def test_analyze_with_the_cuda_backend_probes_statically(api, matmul_source, tmp_path):
    """`analyze` on a "cuda" config: verdicts from the static rules, kernels from the matcher, the reference's report file."""
    cfg_path = _workspace(tmp_path, matmul_source, {"source": "matmul.c", "workdir": "work", "cuda": {"n": 256}})
    rc, out, err = H.cmd_analyze(api, cfg_path)
    assert rc == 0, err
    assert "loops: 12" in out and "gene length: 12" in out and "loop 8: line 25, depth 0 -> candidate [kernel: matmul_nt]" in out
    report = [json.loads(x) for x in (tmp_path / "work" / "probe_report.jsonl").read_text().splitlines()]
    assert [r["id"] for r in report] == list(range(12)) and all(r["verdict"] == "parallelizable" and r["message"] == "" for r in report)
    # a loop the rules reject is listed with its class and drops out of the gene
    poisoned = matmul_source.replace("sum += c[i][i];", "sum += fabs(c[i][i]);")
    (tmp_path / "p").mkdir()
    cfg_path = _workspace(tmp_path / "p", poisoned, {"source": "matmul.c", "workdir": "work", "cuda": {"n": 256}})
    rc, out, _ = H.cmd_analyze(api, cfg_path)
    assert rc == 0 and "gene length: 11" in out
    assert "loop 11: line 31, depth 0 -> rejected [external_call] call to 'fabs' with no acc routine information" in out


def test_sim_runs_write_the_skipped_probe_report(api, matmul_source, tmp_path):
    """commands.cpp:78-97 of the reference: sim runs record one 'probe skipped' row per loop."""
    golden = json.loads((GOLDEN / "tune_sim" / "runs.json").read_text())["m8_t6_seed7"]
    cfg_path = _workspace(tmp_path, matmul_source, golden["config"])
    assert H.cmd_tune(api, cfg_path)[0] == 0
    rows = [json.loads(x) for x in (tmp_path / "work" / "probe_report.jsonl").read_text().splitlines()]
    assert len(rows) == 12 and all(r["message"] == "probe skipped: timings come from a sim model" and r["verdict"] == "parallelizable"
                                   and r["reject_class"] is None and r["timed_out"] is False for r in rows)
    if "probe_report.jsonl" in golden["files"]:
        assert (tmp_path / "work" / "probe_report.jsonl").read_text() == golden["files"]["probe_report.jsonl"]


def test_calibrate_needs_the_cuda_backend_and_a_device(api, matmul_source, tmp_path):
    import torch
    cfg_path = _workspace(tmp_path, matmul_source, {"source": "matmul.c", "workdir": "work", "sim_model": "model.json"})
    rc, _, err = H.cmd_calibrate(api, cfg_path)
    assert rc == 2 and "needs a 'cuda' block" in err
    if not torch.cuda.is_available():
        cfg_path = _workspace(tmp_path, matmul_source, {"source": "matmul.c", "workdir": "work", "cuda": {"n": 64}})
        assert H.cmd_calibrate(api, cfg_path)[0] == 4        # ToolchainMissing: no CPU fallback


@pytest.mark.gpu
def test_calibrate_end_to_end(api, matmul_source, tmp_path):
    """`calibrate`: every feasible genome measured through the evaluator, the reference's model file written; the file
    loads, its optimum is a feasible genome close to the measured one, and `tune --sim` replays it."""
    cfg = {"source": "matmul.c", "workdir": "work", "cuda": {"n": 64, "timeout_s": 20.0, "repetitions": 3, "warmup": 1, "devices": [0, 0]}}
    cfg_path = _workspace(tmp_path, matmul_source, cfg)
    rc, out, err = H.cmd_calibrate(api, cfg_path)
    assert rc == 0, err
    work = tmp_path / "work"
    rep = json.loads((work / "calibration.json").read_text())
    assert rep["feasible_genomes"] == 648 and rep["measured"] + rep["timeouts"] == 648 and rep["measured"] >= 600
    assert capi.plan(rep["cost_best_genome"], 64, capi.F64).feasible
    assert rep["fit_rms_rel_err"] < 0.25
    times = api.model_time_all(work / "calibrated_model.json", 12)
    assert (times > 0).sum() == 648
    lines = (work / "eval_cache.jsonl").read_text().splitlines()
    assert len(lines) == 648
    # the modelled optimum is among the fastest measured genomes
    measured = sorted((json.loads(x)["time_s"], json.loads(x)["genome"]) for x in lines if json.loads(x)["status"] == "measured")
    rank = [g for _, g in measured].index(rep["cost_best_genome"])
    assert rank < 32, (rank, measured[:3])
    rc, out2, _ = H.cmd_calibrate(api, cfg_path)                     # rerun: replayed from the cache, same model
    assert rc == 0 and json.loads((work / "calibration.json").read_text())["cost_best_genome"] == rep["cost_best_genome"]
    rc, out3, err3 = H.cmd_tune(api, cfg_path, seed=1, sim_model=work / "calibrated_model.json")
    assert rc == 0, err3


@pytest.mark.gpu
def test_tune_with_the_cuda_backend_end_to_end(api, matmul_source, tmp_path):
    """The drop-in path: `tune` with a "cuda" block measures real individuals at the fixture size and leaves the
    reference's artifact set; the all-nests-offloaded genome must beat the all-CPU baseline by a wide margin."""
    cfg = {"source": "matmul.c", "workdir": "work", "ga": {"population": 16, "generations": 6, "seed": 3},
           "cuda": {"n": 256, "timeout_s": 5.0, "repetitions": 3, "warmup": 1, "devices": [0, 0]}}
    cfg_path = _workspace(tmp_path, matmul_source, cfg)
    rc, out, err = H.cmd_tune(api, cfg_path)
    assert rc == 0, err
    work = tmp_path / "work"
    summary = json.loads((work / "summary.json").read_text())
    assert summary["speedup"] >= 1.0 and summary["baseline_s"] > 0
    assert capi.plan(summary["best_genome"], 256, capi.F64).feasible
    lines = [json.loads(x) for x in (work / "eval_cache.jsonl").read_text().splitlines()]
    assert len(lines) == summary["distinct_evals"] and {"genome", "status", "time_s", "wall_cost_s"} <= set(lines[0])
    assert any(x["status"] == "compile_error" for x in lines)      # nested-overlap genomes are outcomes, not errors
    best = (work / "best" / "matmul.c").read_text()
    assert best == H.render_variant(api, matmul_source, summary["best_genome"])
    assert H.cmd_report(api, work)[0] == 0
    rc, out2, _ = H.cmd_tune(api, cfg_path)                          # rerun from the cache: nothing is measured again
    assert rc == 0 and ", 0 backend calls" in out2
