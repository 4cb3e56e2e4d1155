"""Static feasibility rules and the kernel matcher against the reference.

Golden: tests/golden/probe_cases.json -- for every synthetic source, the probe report of the reference's
build_candidate_set driving its bundled compiler (probe.cpp:187, tools/mockacc.cpp), and that compiler's verdict and
diagnostics on the reference-rendered variant of every genome (tests/golden/generate_golden.py: gen_probe_cases).
Where oracle/_ref is built and /root/reference is present, the reference's own corpus is probed side by side.
"""
import sys
import json
import re
import tempfile
from pathlib import Path

import pytest

from paper_1806_01430_b200 import hostapi as H

sys.path.insert(0, str(Path(__file__).resolve().parent))
import refapi  # noqa: E402  (test-only loader of the compiled reference)

GOLD = Path(__file__).parent / "golden"
CASES = json.loads((GOLD / "probe_cases.json").read_text())
REF_FIXTURES = Path("/root/reference/proj/fixtures")
MOCKACC = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "mockacc"


def core(message: str) -> list[str]:
    """Diagnostics without the tool prefix: 'what (file: line N)' per line."""
    return [re.sub(r"^mockacc: error: ", "", line) for line in message.splitlines() if line]


@pytest.mark.parametrize("name", sorted(CASES))
def test_probe_report_matches_reference(name):
    case = CASES[name]
    rc, rows = H.probe_source(case["text"], f"{name}.c")
    assert rc == case["rc"]                      # accepted count, or NoCandidates (-9)
    assert len(rows) == len(case["report"])
    for mine, ref in zip(rows, case["report"]):
        assert (mine["id"], mine["line"], mine["verdict"], mine["reject_class"], mine["timed_out"]) == \
               (ref["id"], ref["line"], ref["verdict"], ref["reject_class"], ref["timed_out"])
        assert core(mine["message"]) == core(ref["message"])   # same wording, same variant line numbers


@pytest.mark.parametrize("name", sorted(k for k, v in CASES.items() if v["genomes"]))
def test_every_genome_verdict_matches_reference_compiler(name):
    case = CASES[name]
    for genome, ref in case["genomes"].items():
        ok, diags = H.variant_feasible(case["text"], genome, f"{name}.c")
        assert ok == ref["ok"], (name, genome)
        assert diags == core("\n".join(ref["diagnostics"])), (name, genome)


def test_matrix_app_genomes_match_mockacc_and_the_planner():
    """All 4096 genomes of the matrix application: static rules == mockacc (golden) == mmx_plan().feasible."""
    from paper_1806_01430_b200 import capi
    text = H.strip_directives(H.mine(), (GOLD / "rendered_all_nests.c").read_text())
    verdicts = (GOLD / "feasibility_mockacc.txt").read_text().strip()
    assert len(verdicts) == 4096
    for mask in range(4096):
        g = "".join("1" if (mask >> k) & 1 else "0" for k in range(12))
        ok, _ = H.variant_feasible(text, g, "matmul.c")
        assert ok == (verdicts[mask] == "1"), g
        if mask % 7 == 0:
            assert bool(capi.plan(g, 256, capi.F64).feasible) == ok


def test_kernel_matcher_derives_the_served_catalogue():
    """match_kernels on the application's source == mmx_loop_catalogue (gene, line, depth, nest, induction, kernel)."""
    from paper_1806_01430_b200 import capi
    text = H.strip_directives(H.mine(), (GOLD / "rendered_all_nests.c").read_text())
    m = H.match_kernels(text, "matmul.c")
    served = capi.loop_catalogue()
    assert len(m["loops"]) == len(served) == 12
    for mine, row in zip(m["loops"], served):
        assert (mine["id"], mine["line"], mine["depth"], mine["nest"], mine["var"], mine["kernel"]) == \
               (row["gene"], row["line"], row["depth"], row["nest"], row["induction"], row["kernel"])
        assert mine["why"] == "" and mine["bound"] == "N"
    # producer -> consumer edges the residency planner moves data along (csrc/plan.cpp header)
    assert sorted(map(tuple, m["dataflow"])) == sorted([("a", 0, 4), ("b", 1, 3), ("bt", 3, 4), ("c", 2, 4), ("c", 4, 5)])


MATCH_CASES = {
    # (source, expected [(idiom, kernel)] per loop)
    "float_and_preincrement": (
        "void f(int n) {\n  for (int r = 0; r < n; ++r)\n    for (int s = 0; s < n; s += 1)\n      w[r][s] = (float)(r - s) / n;\n}\n",
        [("fill_affine", "fill2d<init_b>"), ("fill_affine", "fill_row<init_b>")]),
    "zero_literals": (
        "void f(void) {\n  for (int i = 0; i < N; i++) {\n    for (int j = 0; j < N; j++) {\n      c[i][j] = 0.0f;\n    }\n  }\n"
        "  for (int i = 0; i < N; i++)\n    for (int j = 0; j < N; j++)\n      d[i][j] = 0;\n}\n",
        [("fill_zero", "fill2d<zero>"), ("fill_zero", "fill_row<zero>")] * 2),
    "commuted_product": (
        "void f(void) {\n  for (int i = 0; i < N; i++)\n    for (int j = 0; j < N; j++)\n      for (int k = 0; k < N; k++)\n        c[i][j] += q[j][k] * p[i][k];\n}\n",
        [("contraction", "matmul_nt"), ("contraction", "gemv_row"), ("contraction", "dot_rows")]),
    "nn_product_has_no_kernel": (   # b[k][j]: not the K-contiguous form the library serves
        "void f(void) {\n  for (int i = 0; i < N; i++)\n    for (int j = 0; j < N; j++)\n      for (int k = 0; k < N; k++)\n        c[i][j] += a[i][k] * b[k][j];\n}\n",
        [("unknown", "")] * 3),
    "nonzero_fill_and_wrong_bounds": (
        "void f(void) {\n  for (int i = 0; i < N; i++)\n    for (int j = 0; j < N; j++)\n      c[i][j] = 1.0;\n"
        "  for (int i = 1; i < N; i++)\n    for (int j = 0; j < N; j++)\n      c[i][j] = 0.0;\n"
        "  for (int i = 0; i < N; i++)\n    for (int j = 0; j < M; j++)\n      c[i][j] = 0.0;\n}\n",
        [("unknown", "")] * 6),
    "imperfect_nest": (
        "void f(void) {\n  for (int i = 0; i < N; i++) {\n    s += 1.0;\n    for (int j = 0; j < N; j++)\n      c[i][j] = 0.0;\n  }\n"
        "  for (int i = 0; i < N; i++) {\n    for (int j = 0; j < N; j++)\n      c[i][j] = 0.0;\n    for (int j = 0; j < N; j++)\n      d[i][j] = 0.0;\n  }\n}\n",
        [("unknown", "")] * 5),
    "trace_and_offdiagonal": (
        "void f(void) {\n  for (int i = 0; i < N; i++)\n    t += m[i][i];\n  for (int i = 0; i < N; i++)\n    t += m[i][0];\n}\n",
        [("diagonal_sum", "trace_diag"), ("unknown", "")]),
}


@pytest.mark.parametrize("name", sorted(MATCH_CASES))
def test_kernel_matcher_idioms(name):
    text, expected = MATCH_CASES[name]
    got = [(row["idiom"], row["kernel"]) for row in H.match_kernels(text, f"{name}.c")["loops"]]
    assert got == expected
    for row in H.match_kernels(text)["loops"]:
        assert (row["kernel"] == "") == (row["why"] != "")


@pytest.mark.skipif(not (REF_FIXTURES.is_dir() and MOCKACC.exists() and refapi.reference() is not None),
                    reason="needs /root/reference and oracle/_ref (build container only)")
@pytest.mark.parametrize("rel", ["corpus/data_dep.c", "corpus/early_exit.c", "corpus/ext_call.c", "corpus/nested.c", "matmul.c"])
def test_reference_corpus_side_by_side(rel):
    """The reference's own rejection corpus (acceptance.cpp:350-406): its probe with mockacc vs the static rules."""
    text = (REF_FIXTURES / rel).read_text()
    name = Path(rel).name
    rc, rows = H.probe_source(text, name)
    with tempfile.TemporaryDirectory() as td:
        rrc, rrows = refapi.ref_probe_text(text, name, f"{MOCKACC} -acc {{src}} -o {{out}}", td)
    assert rc == rrc and len(rows) == len(rrows)
    for mine, ref in zip(rows, rrows):
        assert {k: mine[k] for k in ("id", "line", "verdict", "reject_class")} == {k: ref[k] for k in ("id", "line", "verdict", "reject_class")}
        assert core(mine["message"]) == [re.sub(r"\(/[^ ]*/", "(", x) for x in core(ref["message"])]
