"""Drop-in proof: the UNMODIFIED reference tuner drives libmmx.so.

`oracle/_ref/drive_reference` links the reference's own `Evaluator` (proj/src/evaluator.cpp:144-292) and `run_ga`
(proj/src/ga.cpp:247-295), compiled from /root/reference by oracle/Makefile, with `acctune::CudaBackend`
(tests/ref_integration/cuda_backend.hpp -- the class INTEGRATION.md section 2 lists, checked verbatim below) which
implements the reference's `EvalBackend` (proj/include/acctune/evaluator.hpp:19-24) over the C ABI.  Nothing of this
repo's host mirror is in that binary.  The binary is built in the build container and travels to the GPU box."""
import json
import re
import subprocess
from pathlib import Path

import pytest

from paper_1806_01430_b200 import capi, hostapi as H

ROOT = Path(__file__).resolve().parent.parent
DRIVER = ROOT / "oracle" / "_ref" / "drive_reference"
GOLDEN = Path(__file__).resolve().parent / "golden"
INNER_GENES = (1, 3, 5, 7, 9, 10)   # loops at depth >= 1


def _source(tmp_path) -> Path:
    src = tmp_path / "matmul.c"
    src.write_text(H.strip_directives(H.mine(), (GOLDEN / "rendered_best.c").read_text()))
    return src


def test_integration_listing_is_the_compiled_binding():
    """INTEGRATION.md section 2 shows exactly the file that is compiled against the reference."""
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```cpp\n(.*?)```", text, flags=re.S)
    header = (ROOT / "tests" / "ref_integration" / "cuda_backend.hpp").read_text()
    assert any(b == header for b in blocks), "INTEGRATION.md section 2 must list tests/ref_integration/cuda_backend.hpp verbatim"


@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref is built only where /root/reference exists")
def test_without_a_device_the_backend_is_toolchain_missing(tmp_path):
    """No CUDA device => mmx_create fails => ToolchainMissing out of the constructor: there is no CPU path to fall to."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    p = subprocess.run([str(DRIVER), str(_source(tmp_path)), str(tmp_path / "w"), "64", "4", "2", "1", "1"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 1 and "no usable CUDA device" in p.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref/drive_reference was not built (needs /root/reference at build time)")
def test_reference_evaluator_and_run_ga_drive_the_cuda_backend(tmp_path):
    work = tmp_path / "work"
    p = subprocess.run([str(DRIVER), str(_source(tmp_path)), str(work), "256", "64", "20", "1", "2"], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    out = json.loads(p.stdout)
    assert out["gene_length"] == 12
    cold, warm = out["cold"], out["warm"]

    # the baseline (all-zero genome) was Measured (ga.cpp:254-258 would have thrown otherwise) on the host clock
    assert cold["baseline_s"] > 0.0
    rows = cold["generations_csv"].splitlines()
    assert rows[0] == "generation,best_time_s,best_speedup,best_genome,mean_fitness,distinct_evals,cache_hits"
    assert len(rows) == 1 + 21 and rows[1].split(",")[3] == "0" * 12

    # every genome the GA asked for went through mmx_measure exactly once; >= 2 calls overlapped, never more than jobs
    c = cold["counters"]
    assert c["backend_calls"] == c["distinct"] == cold["measure_calls"] and c["requests"] == 1 + 64 + 19 * 63
    assert c["cache_hits"] == c["requests"] - c["distinct"]
    assert 2 <= cold["max_in_flight"] <= 2

    # outcomes in the reference's own cache file: infeasible <=> compile_error with time 0 (mockacc.cpp:205-221 semantics)
    lines = [json.loads(l) for l in (work / "eval_cache.jsonl").read_text().splitlines()]
    assert len(lines) == c["distinct"] and len({l["genome"] for l in lines}) == len(lines)
    assert [list(l) for l in lines[:1]] == [["genome", "status", "time_s", "wall_cost_s"]]
    n_bad = 0
    for l in lines:
        feasible = bool(capi.plan(l["genome"], 256, capi.F64).feasible)
        assert (l["status"] == "compile_error") == (not feasible), l
        if not feasible:
            n_bad += 1
            assert l["time_s"] == 0.0
        else:
            assert l["status"] in ("measured", "timeout") and l["time_s"] > 0.0
    assert 0 < n_bad < len(lines)

    # the search found a pattern that offloads the matmul nest as a whole and no inner loop on its own
    best = cold["best_genome"]
    assert best[8] == "1" and not any(best[g] == "1" for g in INNER_GENES), best
    assert capi.plan(best, 256, capi.F64).feasible
    assert cold["baseline_s"] / cold["best_s"] >= 35.0           # the paper's bar, on the fixture size
    assert cold["best_source_has_pragma"]

    # resumed from eval_cache.jsonl: same trajectory, zero backend calls (evaluator.cpp:150-176; test_cli.cpp:371-394)
    assert warm["measure_calls"] == 0 and warm["counters"]["backend_calls"] == 0
    assert warm["counters"]["distinct"] == c["distinct"] and warm["counters"]["requests"] == c["requests"]
    assert warm["generations_csv"] == cold["generations_csv"] and warm["best_genome"] == best

    # error conventions at the boundary
    e = out["errors"]
    assert e["backend_wrong_length"] == "GenomeLengthMismatch" and e["evaluator_wrong_length"] == "GenomeLengthMismatch"
    assert e["infeasible_status"] == "compile_error" and e["infeasible_time_s"] == 0.0
    assert e["all_nests_status"] == "measured" and 0.0 < e["all_nests_time_s"] < 1e-3
    assert out["no_slots"] == "ConfigError"
