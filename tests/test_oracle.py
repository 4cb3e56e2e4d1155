"""The oracle (oracle/matmul_oracle.c) against the reference's own outputs.

Golden values in tests/golden/fixture_n256.json were produced by compiling and running the
UNMODIFIED /root/reference/proj/fixtures/matmul.c (tests/golden/generate_golden.py); where
oracle/_ref/libmatmul_fixture.so is present (it travels with the repo snapshot) the arrays are
also compared element by element.
"""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle import cpu

ROOT = Path(__file__).resolve().parent.parent
FIXTURE_SO = ROOT / "oracle" / "_ref" / "libmatmul_fixture.so"


def test_oracle_matches_fixture_golden(golden):
    g = golden("fixture_n256.json")
    assert g["stdout"] == "checksum 0.000000\n"  # fixtures/matmul.c:34
    app = cpu.App(g["n"]).run()
    assert app.checksum == float.fromhex(g["trace"]) == 0.0
    for name in ("a", "b", "c", "bt"):
        arr = getattr(app, name)
        want = g["arrays"][name]
        assert f"{cpu.fnv1a64(arr):016x}" == want["fnv1a64"], name
        assert float(arr.sum()).hex() == want["sum"]
        assert float(np.abs(arr).sum()).hex() == want["abs_sum"]
        assert float(arr[0, 0]).hex() == want["corner_0_0"]
        assert float(arr[1, 2]).hex() == want["corner_1_2"]
        assert float(arr[-1, -1]).hex() == want["corner_last"]
    # SURVEY appendix A
    assert g["arrays"]["c"]["fnv1a64"] == "463fd603cc85176c"


@pytest.mark.skipif(not FIXTURE_SO.exists(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_compiled_reference_fixture(capfd):
    fx = C.CDLL(str(FIXTURE_SO))
    fx.fixture_run()
    n = fx.fixture_n()
    app = cpu.App(n, threads=3).run()
    for name in ("a", "b", "c", "bt"):
        f = getattr(fx, "fixture_" + name)
        f.restype = C.POINTER(C.c_double)
        ref = np.ctypeslib.as_array(f(), shape=(n, n))
        assert np.array_equal(ref.view(np.uint64), getattr(app, name).view(np.uint64)), name


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 100, 256])
def test_threads_do_not_change_bits(n):
    for dtype in (0, 1):
        one = cpu.App(n, dtype, threads=1).run()
        many = cpu.App(n, dtype, threads=5).run()
        for name in ("a", "b", "c", "bt"):
            assert np.array_equal(getattr(one, name), getattr(many, name))
        assert one.checksum == many.checksum


@pytest.mark.parametrize("n", [4, 64, 256, 512])
def test_closed_form_is_exact_for_powers_of_two(n):
    # all partial sums are dyadic rationals that fit a double
    app = cpu.App(n).run()
    assert np.array_equal(cpu.closed_form_c(n), app.c)
    assert app.checksum == 0.0


def test_closed_form_known_answers():
    lib = cpu.load()
    assert lib.mmo_closed_form(256, 0, 0) == 84.833984375
    assert lib.mmo_closed_form(256, 1, 2) == 84.328125
    assert lib.mmo_closed_form(256, 255, 255) == -169.169921875
    assert lib.mmo_closed_form(1024, 0, 0) == 340.83349609375
    assert lib.mmo_closed_form(1024, 1023, 1023) == -681.16748046875


def test_closed_form_close_for_other_n():
    app = cpu.App(300).run()
    ref = cpu.closed_form_c(300)
    assert not np.array_equal(ref, app.c)  # order matters here (appendix A)
    assert np.abs(ref - app.c).max() < 1e-11


def test_float_flavour_matches_numpy_float32_loop():
    # same program in float: sequential k, separate mul and add, float accumulator
    n = 33
    app = cpu.App(n, 1).run()
    a = ((np.arange(n)[:, None] + np.arange(n)[None, :]).astype(np.float32) / np.float32(n)).astype(np.float32)
    b = ((np.arange(n)[:, None] - np.arange(n)[None, :]).astype(np.float32) / np.float32(n)).astype(np.float32)
    assert np.array_equal(app.a, a) and np.array_equal(app.b, b) and np.array_equal(app.bt, b.T)
    c = np.zeros((n, n), np.float32)
    for k in range(n):
        c = (c + (a[:, k:k + 1] * b.T[:, k][None, :]).astype(np.float32)).astype(np.float32)
    assert np.array_equal(app.c, c)
    s = np.float32(0)
    for i in range(n):
        s = np.float32(s + c[i, i])
    assert app.checksum == float(s)


def test_row_ranges_compose():
    n = 48
    whole = cpu.App(n).run()
    parts = cpu.App(n)
    for nest in range(5):
        parts.run_nest(nest, 0, 20)
        parts.run_nest(nest, 20, n)
    assert np.array_equal(whole.c, parts.c)
    assert parts.run_nest(5) == whole.checksum


def test_time_app_reports_every_nest():
    r = cpu.time_app(64, 0, 2, 16)
    assert set(r["seconds"]) == set(cpu.NESTS) and r["matmul_rows"] == 16
    assert all(v >= 0 for v in r["seconds"].values())
