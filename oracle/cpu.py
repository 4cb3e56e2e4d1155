"""ctypes front end of oracle/libmatmul_oracle.so (matmul_oracle.c) -- TEST INFRASTRUCTURE.

parity: PINNED.  The restatement is checked bit for bit against the reference's own program
(/root/reference/proj/fixtures/matmul.c compiled unmodified into oracle/_ref/libmatmul_fixture.so)
at the fixture size, and against golden hashes generated from it (tests/golden/fixture_n256.json).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
NESTS = ("init_a", "init_b", "zero_c", "transpose", "matmul", "trace")
_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        so = HERE / "libmatmul_oracle.so"
        if not so.exists():
            subprocess.run(["make", "-C", str(HERE), "oracle"], check=True, capture_output=True)
        lib = C.CDLL(str(so))
        lib.mmo_run_nest.restype = C.c_int
        lib.mmo_run_nest.argtypes = [C.c_int] * 6 + [C.c_void_p] * 4
        lib.mmo_trace.restype = C.c_double
        lib.mmo_trace.argtypes = [C.c_int, C.c_int, C.c_void_p]
        lib.mmo_app.restype = C.c_double
        lib.mmo_app.argtypes = [C.c_int] * 3 + [C.c_void_p] * 4
        lib.mmo_closed_form.restype = C.c_double
        lib.mmo_closed_form.argtypes = [C.c_int] * 3
        lib.mmo_closed_form_fill.restype = None
        lib.mmo_closed_form_fill.argtypes = [C.c_int] * 3 + [C.c_void_p]
        lib.mmo_fnv1a64.restype = C.c_uint64
        lib.mmo_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        lib.mmo_time_app.restype = C.c_double
        lib.mmo_time_app.argtypes = [C.c_int] * 4 + [C.POINTER(C.c_double)]
        _lib = lib
    return _lib


def np_dtype(dtype: int):
    return np.float64 if dtype == 0 else np.float32


class App:
    """The program's four arrays plus the nests that act on them (matmul.c:5-32)."""

    def __init__(self, n: int, dtype: int = 0, threads: int = 1):
        self.n, self.dtype, self.threads = n, dtype, threads
        t = np_dtype(dtype)
        # NaN-poisoned so a nest that fails to write shows up
        self.a, self.b, self.c, self.bt = (np.full((n, n), np.nan, dtype=t) for _ in range(4))
        self.checksum = float("nan")

    def _ptrs(self):
        return [x.ctypes.data for x in (self.a, self.b, self.c, self.bt)]

    def run_nest(self, nest: int, r0: int = 0, r1: int | None = None):
        if nest == 5:
            self.checksum = load().mmo_trace(self.dtype, self.n, self.c.ctypes.data)
            return self.checksum
        rc = load().mmo_run_nest(nest, self.dtype, self.n, r0, self.n if r1 is None else r1, self.threads, *self._ptrs())
        assert rc == 0
        return None

    def run(self):
        self.checksum = load().mmo_app(self.dtype, self.n, self.threads, *self._ptrs())
        return self


def closed_form_c(n: int, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """Exact c (FP64) from the closed form, rows [r0, r1) -- no O(N^3) loop."""
    r1 = n if r1 is None else r1
    out = np.zeros((n, n), dtype=np.float64)
    load().mmo_closed_form_fill(n, r0, r1, out.ctypes.data)
    return out[r0:r1]


def fnv1a64(arr: np.ndarray) -> int:
    arr = np.ascontiguousarray(arr)
    return load().mmo_fnv1a64(arr.ctypes.data, arr.nbytes)


def time_app(n: int, dtype: int, threads: int, matmul_rows: int) -> dict:
    secs = (C.c_double * 6)()
    tr = load().mmo_time_app(dtype, n, threads, matmul_rows, secs)
    return {"trace": tr, "seconds": dict(zip(NESTS, list(secs))), "matmul_rows": min(matmul_rows, n)}
