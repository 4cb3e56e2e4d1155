#!/usr/bin/env python
"""Regenerates tests/golden/* from the UNMODIFIED reference (run in the build container only).

Needs /root/reference and `make -C oracle ref` (oracle/_ref/libacctune_ref.so, libmatmul_fixture.so,
mockacc).  Everything written here is an output of the reference's own code:
  fixture_n256.json       arrays left behind by fixtures/matmul.c (hashes, sums, corner values)
  catalogue.json          scan_loops(fixtures/matmul.c): id, line, depth of every `for`
  feasibility_mockacc.txt mockacc's accept/reject verdict for all 4096 genomes of matmul.c
  model_times_*.npy       model_time() of every genome of the three fixture cost models
  ga_runs.json            run_ga trajectories (generations.csv text, best, counters)
  ga_operators.json       Rng draws, init_population, breed / roulette / mutate / crossover,
                          fitness_from_time, assign_fitness vectors
  eval_cache_sample.jsonl the first lines Evaluator appends to its cache file
  rendered_best.c         render_variant(matmul.c, "100000000000")
  models/*.json           copies of fixtures/models/*.json (input data of the runs above)
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = Path("/root/reference/proj")
REFLIB = ROOT / "oracle" / "_ref"
FIXTURE_SRC = REF / "fixtures" / "matmul.c"

sys.path.insert(0, str(ROOT))
from oracle import cpu  # noqa: E402  (only for the FNV helper)


class RefOutcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("time_s", C.c_double), ("wall_cost_s", C.c_double)]


def load_ref() -> C.CDLL:
    lib = C.CDLL(str(REFLIB / "libacctune_ref.so"))
    lib.ref_last_error.restype = C.c_char_p
    return lib


def bits_of(s: str):
    arr = (C.c_uint8 * len(s))(*[int(ch) for ch in s])
    return arr


def str_of(arr, n) -> str:
    return "".join(str(int(arr[i])) for i in range(n))


def gen_fixture():
    fx = C.CDLL(str(REFLIB / "libmatmul_fixture.so"))
    # the program prints its checksum line; capture it through a child process to keep stdout clean
    out = subprocess.run(
        [sys.executable, "-c",
         f"import ctypes; fx = ctypes.CDLL('{REFLIB / 'libmatmul_fixture.so'}'); fx.fixture_run()"],
        capture_output=True, text=True, check=True).stdout
    fx.fixture_run.restype = C.c_int
    # silence our own copy of the run
    devnull = os.open(os.devnull, os.O_WRONLY)
    saved = os.dup(1)
    os.dup2(devnull, 1)
    try:
        fx.fixture_run()
    finally:
        os.dup2(saved, 1)
        os.close(devnull)
    n = fx.fixture_n()
    res = {"n": n, "stdout": out, "source": str(FIXTURE_SRC), "arrays": {}}
    for name in ("a", "b", "c", "bt"):
        f = getattr(fx, "fixture_" + name)
        f.restype = C.POINTER(C.c_double)
        arr = np.ctypeslib.as_array(f(), shape=(n, n)).copy()
        res["arrays"][name] = {
            "fnv1a64": f"{cpu.fnv1a64(arr):016x}",
            "sum": float(arr.sum()).hex(),
            "abs_sum": float(np.abs(arr).sum()).hex(),
            "corner_0_0": float(arr[0, 0]).hex(),
            "corner_1_2": float(arr[1, 2]).hex(),
            "corner_last": float(arr[n - 1, n - 1]).hex(),
        }
    res["trace"] = float(np.trace(np.ctypeslib.as_array(fx.fixture_c(), shape=(n, n)))).hex()
    (HERE / "fixture_n256.json").write_text(json.dumps(res, indent=1) + "\n")


def gen_catalogue(lib):
    buf = C.create_string_buffer(4096)
    rc = lib.ref_scan_loops(str(FIXTURE_SRC).encode(), buf, C.c_size_t(4096))
    assert rc > 0, lib.ref_last_error()
    rows = [dict(zip(("id", "line", "depth"), map(int, line.split(",")))) for line in buf.value.decode().splitlines()]
    (HERE / "catalogue.json").write_text(json.dumps(rows, indent=1) + "\n")


def gen_feasibility(lib):
    """mockacc verdict per genome; index = sum(bit_k << k) (bit k = gene k)."""
    verdict = []
    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "matmul.c"
        exe = Path(td) / "out.bin"
        buf = C.create_string_buffer(1 << 16)
        for mask in range(1 << 12):
            s = "".join("1" if (mask >> k) & 1 else "0" for k in range(12))
            n = lib.ref_render_variant(str(FIXTURE_SRC).encode(), bits_of(s), C.c_size_t(12), buf, C.c_size_t(1 << 16))
            assert n > 0
            src.write_bytes(buf.value)
            rc = subprocess.run([str(REFLIB / "mockacc"), "-acc", str(src), "-o", str(exe)], capture_output=True).returncode
            verdict.append("1" if rc == 0 else "0")
    (HERE / "feasibility_mockacc.txt").write_text("".join(verdict) + "\n")
    print("feasible genomes:", verdict.count("1"))


def gen_model_times(lib):
    for name, a in (("matrix12", 12), ("separable", 8), ("coupled", 10)):
        path = REF / "fixtures" / "models" / f"{name}.json"
        times = np.zeros(1 << a, dtype=np.float64)
        rc = lib.ref_model_time_all(str(path).encode(), times.ctypes.data_as(C.POINTER(C.c_double)), C.c_size_t(times.size))
        assert rc == a, (rc, lib.ref_last_error())
        np.save(HERE / f"model_times_{name}.npy", times)
        best = (C.c_uint8 * a)()
        t = C.c_double()
        assert lib.ref_exhaustive_best(str(path).encode(), best, C.c_size_t(a), C.byref(t)) == 0
        (HERE / f"model_best_{name}.json").write_text(json.dumps({"genome": str_of(best, a), "time_s": t.value.hex()}) + "\n")


def run_ga(lib, model: str, source, m, t, pc, pm, elite, seed, jobs=1, cache=None):
    a = {"matrix12": 12, "separable": 8, "coupled": 10}[model]
    path = REF / "fixtures" / "models" / f"{model}.json"
    csv = C.create_string_buffer(1 << 16)
    best = (C.c_uint8 * a)()
    best_s, base_s, elapsed = C.c_double(), C.c_double(), C.c_double()
    counters = (C.c_uint64 * 4)()
    rc = lib.ref_run_ga_sim(str(path).encode(), str(source).encode() if source else None, m, t, C.c_double(pc),
                            C.c_double(pm), elite, C.c_uint64(seed), jobs, str(cache).encode() if cache else None,
                            csv, C.c_size_t(1 << 16), best, C.byref(best_s), C.byref(base_s), counters, C.byref(elapsed))
    assert rc > 0, (rc, lib.ref_last_error())
    return {
        "model": model, "source": "fixtures/matmul.c" if source else None, "population": m, "generations": t,
        "crossover_rate": pc, "mutation_rate": pm, "elite_count": elite, "seed": seed,
        "csv": csv.value.decode(), "best_genome": str_of(best, a), "best_s": best_s.value.hex(),
        "baseline_s": base_s.value.hex(),
        "counters": {"requests": counters[0], "distinct": counters[1], "cache_hits": counters[2], "backend_calls": counters[3]},
        "elapsed_s": elapsed.value.hex(),
    }


def gen_ga_runs(lib):
    runs = []
    runs.append(run_ga(lib, "matrix12", FIXTURE_SRC, 12, 12, 0.9, 0.05, 1, 1))
    runs.append(run_ga(lib, "matrix12", FIXTURE_SRC, 64, 40, 0.9, 0.05, 1, 1))
    for seed in (2, 3, 7, 20):
        runs.append(run_ga(lib, "matrix12", FIXTURE_SRC, 12, 12, 0.9, 0.05, 1, seed))
    for model in ("separable", "coupled"):
        for seed in (1, 2, 5):
            runs.append(run_ga(lib, model, None, 12, 12, 0.9, 0.05, 1, seed))
    runs.append(run_ga(lib, "coupled", None, 9, 7, 0.6, 0.2, 3, 11))   # odd offspring count, elite 3
    runs.append(run_ga(lib, "separable", None, 2, 3, 1.0, 1.0, 1, 4))  # smallest legal population
    runs.append(run_ga(lib, "matrix12", FIXTURE_SRC, 16, 5, 0.0, 0.0, 1, 9))  # no crossover, no mutation
    (HERE / "ga_runs.json").write_text(json.dumps(runs, indent=1) + "\n")
    with tempfile.TemporaryDirectory() as td:
        cache = Path(td) / "cache" / "eval_cache.jsonl"
        run_ga(lib, "matrix12", FIXTURE_SRC, 12, 12, 0.9, 0.05, 1, 1, cache=cache)
        lines = cache.read_text().splitlines()
        (HERE / "eval_cache_sample.jsonl").write_text("\n".join(lines[:16]) + "\n")


def gen_operators(lib):
    out = {}
    # Rng helpers (rng.hpp:13-31)
    rng = {}
    for seed in (1, 2, 12345):
        vals = (C.c_double * 16)()
        raws = (C.c_uint64 * 16)()
        entry = {}
        lib.ref_rng_draws(C.c_uint64(seed), 3, C.c_uint64(0), C.c_size_t(16), vals, raws)
        entry["raw"] = [int(x) for x in raws]
        lib.ref_rng_draws(C.c_uint64(seed), 0, C.c_uint64(0), C.c_size_t(16), vals, raws)
        entry["bit"] = [int(x) for x in vals]
        lib.ref_rng_draws(C.c_uint64(seed), 1, C.c_uint64(0), C.c_size_t(16), vals, raws)
        entry["real01"] = [float(x).hex() for x in vals]
        lib.ref_rng_draws(C.c_uint64(seed), 2, C.c_uint64(11), C.c_size_t(16), vals, raws)
        entry["index11"] = [int(x) for x in vals]
        rng[str(seed)] = entry
    out["rng"] = rng

    # init_population (ga.cpp:34-44)
    pops = []
    for a, m, seed in ((12, 8, 1), (12, 12, 1), (8, 5, 3), (1, 4, 2)):
        bits = (C.c_uint8 * (a * m))()
        assert lib.ref_init_population(C.c_size_t(a), m, C.c_uint64(seed), bits) == 0
        pops.append({"a": a, "m": m, "seed": seed, "genomes": [str_of(bits[i * a:(i + 1) * a], a) for i in range(m)]})
    out["init_population"] = pops

    # fitness_from_time (ga.cpp:29-32)
    fit = []
    for t in (4.0, 92.27, 2.43, 0.00243, 1.0, 1e-9, 120.0):
        f = C.c_double()
        assert lib.ref_fitness_from_time(C.c_double(t), C.byref(f)) == 0
        fit.append({"t": float(t).hex(), "fitness": f.value.hex()})
    f = C.c_double()
    out["fitness_from_time"] = fit
    out["fitness_nonpositive_rc"] = [lib.ref_fitness_from_time(C.c_double(t), C.byref(f)) for t in (0.0, -1.0, float("nan"))]

    # assign_fitness (ga.cpp:46-58): status 1 measured, 2 failed
    cases = []
    for status, times in (([1, 2, 1, 2], [4.0, 0.0, 0.25, 0.0]), ([2, 2, 2], [0.0, 0.0, 0.0]), ([1, 1], [1.0, 9.0])):
        m = len(status)
        fo = (C.c_double * m)()
        assert lib.ref_assign_fitness((C.c_int32 * m)(*status), (C.c_double * m)(*times), C.c_size_t(m), fo) == 0
        cases.append({"status": status, "time_s": [float(x).hex() for x in times], "fitness": [float(x).hex() for x in fo]})
    out["assign_fitness"] = cases

    # roulette_select (ga.cpp:60-83)
    rl = []
    for fitness, count, seed in (([1.0, 2.0, 3.0, 4.0], 24, 1), ([0.5, 0.0, 0.5], 16, 7), ([1e-3, 10.0, 1e-3, 3.3], 32, 5)):
        m = len(fitness)
        picks = (C.c_int32 * count)()
        assert lib.ref_roulette((C.c_double * m)(*fitness), C.c_size_t(m), C.c_size_t(count), C.c_uint64(seed), picks) == 0
        rl.append({"fitness": [float(x).hex() for x in fitness], "count": count, "seed": seed, "picks": [int(x) for x in picks]})
    out["roulette_zero_total_rc"] = lib.ref_roulette((C.c_double * 2)(0.0, 0.0), C.c_size_t(2), C.c_size_t(1), C.c_uint64(1), (C.c_int32 * 1)())
    out["roulette"] = rl

    # mutate (ga.cpp:85-92) and one_point_crossover (ga.cpp:94-120)
    mut = []
    for g, pm, seed in (("000000000000", 0.5, 1), ("101010101010", 0.05, 2), ("1111", 1.0, 3), ("1111", 0.0, 3)):
        o = (C.c_uint8 * len(g))()
        assert lib.ref_mutate(bits_of(g), C.c_size_t(len(g)), C.c_double(pm), C.c_uint64(seed), o) == 0
        mut.append({"genome": g, "pm": pm, "seed": seed, "out": str_of(o, len(g))})
    out["mutate"] = mut
    xo = []
    for p1, p2, seed in (("000000000000", "111111111111", 1), ("101010101010", "010101010101", 2), ("00", "11", 3), ("0110", "1001", 8)):
        c1, c2 = (C.c_uint8 * len(p1))(), (C.c_uint8 * len(p1))()
        assert lib.ref_one_point_crossover(bits_of(p1), bits_of(p2), C.c_size_t(len(p1)), C.c_uint64(seed), c1, c2) == 0
        xo.append({"p1": p1, "p2": p2, "seed": seed, "c1": str_of(c1, len(p1)), "c2": str_of(c2, len(p1))})
    out["one_point_crossover"] = xo

    # breed (ga.cpp:139-176)
    br = []
    rs = np.random.RandomState(0)
    for a, m, pc, pm, elite, seed, skip in ((12, 12, 0.9, 0.05, 1, 1, 144), (12, 9, 0.5, 0.3, 2, 4, 0), (6, 4, 1.0, 0.0, 1, 2, 5),
                                            (12, 8, 0.9, 0.05, 1, 3, 0)):
        genomes = ["".join(str(x) for x in rs.randint(0, 2, a)) for _ in range(m)]
        fitness = [float(x) for x in rs.rand(m) * 10]
        if m == 8:  # ties in fitness: elite must be the lexicographically smaller genome
            fitness = [1.0] * m
        flat = (C.c_uint8 * (a * m))(*[int(ch) for g in genomes for ch in g])
        nxt = (C.c_uint8 * (a * m))()
        rc = lib.ref_breed(flat, (C.c_double * m)(*fitness), C.c_size_t(m), C.c_size_t(a), C.c_double(pc), C.c_double(pm),
                           elite, C.c_uint64(seed), C.c_uint64(skip), nxt)
        assert rc == 0, lib.ref_last_error()
        br.append({"a": a, "m": m, "pc": pc, "pm": pm, "elite": elite, "seed": seed, "skip": skip, "genomes": genomes,
                   "fitness": [x.hex() for x in fitness], "next": [str_of(nxt[i * a:(i + 1) * a], a) for i in range(m)]})
    out["breed"] = br
    (HERE / "ga_operators.json").write_text(json.dumps(out, indent=1) + "\n")


def gen_rendered(lib):
    buf = C.create_string_buffer(1 << 16)
    n = lib.ref_render_variant(str(FIXTURE_SRC).encode(), bits_of("100000000000"), C.c_size_t(12), buf, C.c_size_t(1 << 16))
    assert n > 0
    (HERE / "rendered_best.c").write_bytes(buf.value)
    n = lib.ref_render_variant(str(FIXTURE_SRC).encode(), bits_of("101010101001"), C.c_size_t(12), buf, C.c_size_t(1 << 16))
    (HERE / "rendered_all_nests.c").write_bytes(buf.value)


# Synthetic sources written for this repo: one per accept/reject rule and its edge cases.  The golden verdicts come from the
# reference's own probe (build_candidate_set, probe.cpp:187) driving the reference's bundled compiler (tools/mockacc.cpp), and
# from that compiler run on the reference-rendered variant of every genome.
PROBE_CASES = {
    "dependence": "void f(double* a, double* b, double* xa, int n) {\n  for (int i = 1; i < n; i++)\n    a[i] = a[i - 1] + 1.0;\n"
                  "  for (int i = 0; i < n - 1; i++)\n    a[i] = b[i + 1] * 2.0;\n  for (int i = 1; i < n; i++)\n    b[i] += b[i - 1];\n"
                  "  for (int i = 2; i < n; i++)\n    xa[i] = a[i-2] * 2;\n  for (int i = 1; i < n; i++) {\n    if (a[i] == a[i - 1]) b[i] = 0.0;\n  }\n"
                  "  for (int i = 1; i < n; i++) {\n    b[i] = 1.0;\n    a[i] = b[i] + a[i + 10];\n  }\n}\n",
    "calls": "#include <math.h>\n#define MAX(x, y) ((x) > (y) ? (x) : (y))\nvoid g(double* a, double* b, int n) {\n"
             "  for (int i = 0; i < n; i++)\n    a[i] = sqrt(b[i]);\n  for (int i = 0; i < n; i++)\n    a[i] = (double)(i) * sizeof(double);\n"
             "  for (int i = 0; i < n; i++)\n    a[i] = MAX(a[i], b[i]);\n  for (int i = 0; i < n; i++) {\n    /* log(a[i]) would be a call */\n    a[i] = b[i]; // exp(x)\n  }\n"
             "  for (int i = 0; i < n; i++) {\n    const char* s = \"f(x)\";\n    a[i] = s[0];\n  }\n  for (int i = 0; i < n; i++)\n    a[i] = b [i] + fabs  (b[i]);\n}\n",
    "exits": "int h(double* a, int n, int mode) {\n  for (int i = 0; i < n; i++) {\n    switch (mode) {\n      case 0: a[i] = 1.0; break;\n      default: a[i] = 2.0;\n    }\n  }\n"
             "  for (int i = 0; i < n; i++) {\n    if (a[i] < 0.0) return i;\n  }\n  for (int i = 0; i < n; i++) {\n    if (a[i] > 9.0) goto out;\n  }\n"
             "  for (int i = 0; i < n; i++) {\n    double breakfast = a[i]; /* break */\n    a[i] = breakfast * 2.0; // return\n  }\nout:\n  return -1;\n}\n",
    "preannotated": "void k(double* a, double* b, int n, int m) {\n  #  pragma   acc   kernels\n  for (int i = 0; i < n; i++) {\n    for (int j = 0; j < m; j++)\n      b[i * m + j] = a[i * m + j];\n  }\n"
                    "  #pragma acc kernelsx\n  for (int i = 0; i < n; i++) {\n    for (int j = 0; j < m; j++)\n      a[i * m + j] = 0.0;\n  }\n"
                    "  for (int i = 0; i < n; i++) {\n    #pragma acc kernels loop independent\n    #pragma acc kernels\n    for (int j = 0; j < m; j++)\n      a[i * m + j] += 1.0;\n  }\n}\n",
    "triple": "void t(double* a, int n) {\n  for (int i = 0; i < n; i++)\n    for (int j = 0; j < n; j++) {\n      for (int k = 0; k < n; k++)\n        a[i] += 1.0;\n      for (int l = 0; l < n; l++)\n        a[j] += 2.0;\n    }\n}\n",
    "poisoned": "#include <stdio.h>\nvoid p(double* a, int n) {\n#pragma acc kernels\n  for (int i = 0; i < n; i++)\n    printf(\"%f\\n\", a[i]);\n  for (int i = 1; i < n; i++)\n    a[i] = a[i - 1];\n  for (int i = 0; i < n; i++)\n    a[i] = 0.0;\n}\n",
    "all_rejected": "#include <stdlib.h>\nvoid r(double* a, int n) {\n  for (int i = 0; i < n; i++)\n    a[i] = rand();\n  for (int i = 0; i < n; i++) {\n    if (a[i] > 1.0) break;\n  }\n}\n",
    "no_loops": "int main(void) { return 0; }\n",
}


def gen_probe_cases(lib):
    import re
    out = {}
    mock = REFLIB / "mockacc"
    for name, text in PROBE_CASES.items():
        with tempfile.TemporaryDirectory() as td:
            buf = C.create_string_buffer(1 << 16)
            rc = lib.ref_probe_text(text.encode(), f"{name}.c".encode(), f"{mock} -acc {{src}} -o {{out}}".encode(), td.encode(), buf, C.c_size_t(1 << 16))
            rows = [json.loads(line) for line in buf.value.decode().splitlines() if line]
            for r in rows:   # keep the diagnostics, drop the temporary directory from their location
                r["message"] = re.sub(r"\(/[^ ]*/probe/loop_\d+/", "(", r["message"])
            # every genome over all scanned loops: does the reference's compiler accept the reference-rendered variant?
            a = len(rows)
            genomes = {}
            src, exe = Path(td) / f"{name}.c", Path(td) / "out.bin"
            rbuf = C.create_string_buffer(1 << 16)
            for mask in range(1 << a if 0 < a <= 7 else 0):
                g = "".join("1" if (mask >> k) & 1 else "0" for k in range(a))
                assert lib.ref_render_text(text.encode(), bits_of(g), C.c_size_t(a), rbuf, C.c_size_t(1 << 16)) > 0
                src.write_bytes(rbuf.value)
                proc = subprocess.run([str(mock), "-acc", str(src), "-o", str(exe)], capture_output=True, text=True)
                genomes[g] = {"ok": proc.returncode == 0,
                              "diagnostics": [re.sub(r"\(/[^ ]*/", "(", line) for line in proc.stderr.splitlines()]}
            out[name] = {"text": text, "rc": rc, "report": rows, "genomes": genomes}
    (HERE / "probe_cases.json").write_text(json.dumps(out, indent=1) + "\n")
    print("probe cases:", {k: v["rc"] for k, v in out.items()})


SCAN_CASES = {
    "braceless_nest": "void f(int n, double a[8][8]) {\n  int i, j;\n  for (i = 0; i < n; i++)\n    for (j = 0; j < n; j++)\n      a[i][j] = 0.0;\n}\n",
    "comments_and_strings": "/* for (;;) in a comment */\nint g(void) {\n  const char* s = \"for (x) { \\\" }\";  // for (y)\n  char c = '{';\n  int k = 0;\n\tfor (int i = 0; i < 3; ++i) { k += i; }\n  return k + (c == s[0]);\n}\n",
    "preprocessor": "#define LOOP for (int q = 0; q < 4; ++q) \\\n    do_it(q);\n#include <stdio.h>\nvoid h(void) {\n  LOOP\n  for (int i = 0; i < 2; ++i)\n    ;\n}\n",
    "if_else_do_while": "void k(int n) {\n  if (n > 0)\n    for (int i = 0; i < n; ++i) n--;\n  else {\n    do {\n      for (int j = 0; j < 3; ++j) { while (n < 0) for (int z = 0; z < 1; ++z) n++; }\n    } while (n < 10);\n  }\n  switch (n) { case 1: for (;;) break; default: break; }\n}\n",
    "same_line_and_struct": "struct P { int x; } p = { 1 };\nvoid m(int n) { for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) p.x += i * j; }\nint arr[] = { 1, 2, 3 };\nvoid w(void) {\n    for (int forty = 0; forty < 2; ++forty) { int format = forty; (void)format; }\n}\n",
    "no_loops": "int main(void) { return 0; }\n",
}


def gen_scan_cases(lib):
    """Synthetic sources (written for this repo) scanned and rendered by the reference."""
    out = {}
    for name, text in SCAN_CASES.items():
        buf = C.create_string_buffer(1 << 14)
        rc = lib.ref_scan_text(text.encode(), buf, C.c_size_t(1 << 14))
        assert rc >= 0, (name, lib.ref_last_error())
        rows = [list(map(int, line.split(","))) for line in buf.value.decode().splitlines()]
        n = len(rows)
        renders = {}
        for genome in {"1" * n, ("10" * n)[:n], ("01" * n)[:n]} if n else set():
            rbuf = C.create_string_buffer(1 << 14)
            assert lib.ref_render_text(text.encode(), bits_of(genome), C.c_size_t(n), rbuf, C.c_size_t(1 << 14)) > 0
            renders[genome] = rbuf.value.decode()
        out[name] = {"text": text, "rows": rows, "renders": renders}
    (HERE / "scan_cases.json").write_text(json.dumps(out, indent=1) + "\n")


def gen_tune_runs(lib):
    """Artifact sets of the reference's cmd_tune on fixtures/matmul.c + models/matrix12.json (sim backend)."""
    dst = HERE / "tune_sim"
    dst.mkdir(exist_ok=True)
    runs = {"default_seed1": {"seed": 1}, "m8_t6_seed7": {"population": 8, "generations": 6, "seed": 7},
            "m64_t40_seed1": {"population": 64, "generations": 40, "seed": 1}}
    index = {}
    for name, ga in runs.items():
        with tempfile.TemporaryDirectory() as tmp:
            tmp = Path(tmp)
            (tmp / "matmul.c").write_bytes(FIXTURE_SRC.read_bytes())
            (tmp / "model.json").write_bytes((REF / "fixtures" / "models" / "matrix12.json").read_bytes())
            cfg = {"source": "matmul.c", "workdir": "work", "jobs": 1, "ga": ga, "sim_model": "model.json"}
            (tmp / "cfg.json").write_text(json.dumps(cfg))
            out, err = C.create_string_buffer(1 << 14), C.create_string_buffer(1 << 14)
            rc = lib.ref_cmd_tune(str(tmp / "cfg.json").encode(), 0, C.c_uint64(0), out, C.c_size_t(1 << 14), err, C.c_size_t(1 << 14))
            assert rc == 0, err.value
            rout, rerr = C.create_string_buffer(1 << 14), C.create_string_buffer(1 << 14)
            assert lib.ref_cmd_report(str(tmp / "work").encode(), rout, C.c_size_t(1 << 14), rerr, C.c_size_t(1 << 14)) == 0
            files = {}
            for rel in ("config.resolved.json", "generations.csv", "summary.json", "eval_cache.jsonl", "probe_report.jsonl"):
                files[rel] = (tmp / "work" / rel).read_text().replace(str(tmp), "@TMP@")
            best = (tmp / "work" / "best" / "matmul.c").read_text()
            index[name] = {"config": cfg, "stdout": out.value.decode().replace(str(tmp), "@TMP@"), "report_stdout": rout.value.decode(),
                           "files": files, "best_genome_render_sha": fnv(best), "best_is_render_of": json.loads(files["summary.json"])["best_genome"]}
    (dst / "runs.json").write_text(json.dumps(index, indent=1) + "\n")


def fnv(text: str) -> str:
    h = 0xcbf29ce484222325
    for b in text.encode():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def gen_models():
    """The three cost-model fixtures are input DATA of the golden runs: keep a copy beside them."""
    dst = HERE / "models"
    dst.mkdir(exist_ok=True)
    for name in ("matrix12", "separable", "coupled"):
        (dst / f"{name}.json").write_bytes((REF / "fixtures" / "models" / f"{name}.json").read_bytes())


def main():
    if not REF.is_dir():
        sys.exit("needs /root/reference (build container only)")
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "-j8", "oracle", "ref"], check=True, capture_output=True)
    lib = load_ref()
    gen_fixture()
    gen_models()
    gen_catalogue(lib)
    gen_model_times(lib)
    gen_ga_runs(lib)
    gen_operators(lib)
    gen_rendered(lib)
    gen_feasibility(lib)
    gen_scan_cases(lib)
    gen_probe_cases(lib)
    gen_tune_runs(lib)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
