"""ctypes binding of include/mmx.h -- the stub a Python caller of the C ABI uses.

This is plumbing for tests, bench.py and __graft_entry__: the product is libmmx.so.  Loading
fails loudly when the library has not been built; creating a context fails loudly
(`MmxError` with code MMX_E_NODEVICE) when there is no CUDA device -- there is no CPU path
behind a GPU-mapped loop.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "lib"

GENE_LENGTH = 12
NUM_NESTS = 6
NUM_ARRAYS = 4
MAX_PLAN_STEPS = 32

OK, E_INVALID, E_LENGTH, E_NODEVICE, E_NOMEM, E_CUDA, E_STATE = 0, -1, -2, -3, -4, -5, -6
MEASURED, COMPILE_ERROR, RUNTIME_ERROR, TIMEOUT = 0, 1, 2, 3
STATUS_NAMES = ("measured", "compile_error", "runtime_error", "timeout")  # evaluation.cpp:5-25
F64, F32 = 0, 1
FAST, STRICT = 0, 1
ARRAY_A, ARRAY_B, ARRAY_C, ARRAY_BT = range(4)
NEST_NAMES = ("init_a", "init_b", "zero_c", "transpose", "matmul", "trace")
MODE_CPU, MODE_GPU_NEST, MODE_GPU_INNER, MODE_GPU_INNER2 = range(4)
STEP_H2D, STEP_D2H, STEP_D2H_DIAG, STEP_CPU, STEP_GPU, STEP_D2H_SUM, STEP_H2D_DIAG = range(7)
STEP_NAMES = ("h2d", "d2h", "d2h_diag", "cpu", "gpu", "d2h_sum", "h2d_diag")
PEAK_COPY, PEAK_WRITE, PEAK_FP64_FMA, PEAK_FP64_DMMA, PEAK_FP32_FMA, PEAK_READ, PEAK_UMMA_I8, PEAK_UMMA_TF32, PEAK_UMMA_BF16 = range(9)


class Config(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("n", C.c_int32), ("dtype", C.c_int32), ("numerics", C.c_int32),
        ("timeout_s", C.c_double), ("repetitions", C.c_int32), ("num_slots", C.c_int32),
        ("devices", C.POINTER(C.c_int32)), ("host_threads", C.c_int32), ("launch_batching", C.c_int32),
        ("matmul_variant", C.c_int32), ("warmup", C.c_int32),
        ("pin_host", C.c_int32), ("host_core_first", C.c_int32), ("host_core_count", C.c_int32),
        ("early_timeout", C.c_int32),
    ]


class Outcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("time_s", C.c_double), ("wall_cost_s", C.c_double)]

    def as_tuple(self):
        return (self.status, self.time_s, self.wall_cost_s)


class RunStats(C.Structure):
    _fields_ = [
        ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("graph_launches", C.c_uint64), ("checksum", C.c_double), ("gpu_ms", C.c_double),
        ("host_s", C.c_double), ("nest_s", C.c_double * NUM_NESTS),
        ("host_loadavg", C.c_double), ("host_cpus", C.c_int32), ("host_first_cpu", C.c_int32),
    ]


class PlanStep(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nest", C.c_int32), ("array", C.c_int32), ("mode", C.c_int32),
                ("bytes", C.c_uint64), ("launches", C.c_uint64)]


class PlanInfo(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32), ("conflict_nest", C.c_int32), ("modes", C.c_int32 * NUM_NESTS),
        ("num_steps", C.c_int32), ("steps", PlanStep * MAX_PLAN_STEPS),
        ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("h2d_lower_bound", C.c_uint64), ("d2h_lower_bound", C.c_uint64),
    ]


class LoopInfo(C.Structure):
    _fields_ = [("gene", C.c_int32), ("line", C.c_int32), ("depth", C.c_int32), ("nest", C.c_int32),
                ("induction", C.c_char_p), ("kernel", C.c_char_p)]


class ShardHandle(C.Structure):
    _fields_ = [("mem", C.c_ubyte * 64), ("event", C.c_ubyte * 64)]


class ShardStats(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("row0", C.c_int32), ("rows", C.c_int32),
                ("gpu_ms", C.c_double), ("exchange_ms", C.c_double), ("matmul_ms", C.c_double),
                ("peer_bytes", C.c_uint64), ("partial_trace", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class MmxError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"mmx error {code}: {message}")
        self.code = code


# Every symbol include/mmx.h declares, with its signature (tests check the header against this).
_SIGNATURES = {
    "mmx_loop_catalogue": (C.c_int, [C.POINTER(LoopInfo), C.c_size_t]),
    "mmx_plan": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.POINTER(PlanInfo)]),
    "mmx_default_config": (None, [C.POINTER(Config)]),
    "mmx_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "mmx_destroy": (None, [C.c_void_p]),
    "mmx_gene_length": (C.c_size_t, [C.c_void_p]),
    "mmx_num_slots": (C.c_int, [C.c_void_p]),
    "mmx_last_error": (C.c_char_p, [C.c_void_p]),
    "mmx_measure": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.POINTER(Outcome)]),
    "mmx_measure_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.POINTER(Outcome)]),
    "mmx_last_stats": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(RunStats)]),
    "mmx_fetch_array": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "mmx_fetch_rows": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "mmx_upload_array": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "mmx_run_loop": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "mmx_run_loop_rows": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "mmx_device_ptr": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "mmx_gene8_form": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int32)]),
    "mmx_gene8_pick_form": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "mmx_time_gene8_contraction": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "mmx_shard_run_local": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int, C.POINTER(ShardStats), C.POINTER(C.c_double)]),
    "mmx_shard_export": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(ShardHandle)]),
    "mmx_shard_bind": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(ShardHandle), C.POINTER(C.c_int32)]),
    "mmx_shard_phase1": (C.c_int, [C.c_void_p, C.c_int]),
    "mmx_shard_phase2": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(ShardStats)]),
    "mmx_time_loop": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "mmx_peak_probe": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double)]),
}

_lib = None


def lib_path() -> Path:
    return LIB_DIR / "libmmx.so"


def load() -> C.CDLL:
    """Load libmmx.so (no CUDA call happens at load time)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not path.exists():
            raise FileNotFoundError(
                f"{path} is missing: build it with `python -m paper_1806_01430_b200.build` "
                "(there is no fallback implementation)")
        lib = C.CDLL(str(path))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def genome_bits(genome) -> np.ndarray:
    """'101000011000' / iterable of 0/1 -> uint8 array (Genome::bits(), genome.hpp:55)."""
    if isinstance(genome, str):
        if any(ch not in "01" for ch in genome):
            raise ValueError(f"genome string must be over {{0,1}}: {genome}")
        return np.frombuffer(genome.encode(), dtype=np.uint8) - ord("0")
    return np.ascontiguousarray(np.asarray(genome, dtype=np.uint8))


def loop_catalogue() -> list[dict]:
    rows = (LoopInfo * GENE_LENGTH)()
    n = load().mmx_loop_catalogue(rows, GENE_LENGTH)
    return [dict(gene=r.gene, line=r.line, depth=r.depth, nest=r.nest, induction=r.induction.decode(),
                 kernel=r.kernel.decode()) for r in rows[:n]]


def plan(genome, n: int, dtype: int = F64) -> PlanInfo:
    bits = genome_bits(genome)
    info = PlanInfo()
    rc = load().mmx_plan(bits.ctypes.data, bits.size, n, dtype, C.byref(info))
    if rc != OK:
        raise MmxError(rc, "mmx_plan")
    return info


def plan_steps(info: PlanInfo) -> list[tuple]:
    """[(step name, nest name | array index | None, mode, bytes, launches)]"""
    out = []
    for s in info.steps[: info.num_steps]:
        what = NEST_NAMES[s.nest] if s.nest >= 0 else (s.array if s.array >= 0 else None)
        out.append((STEP_NAMES[s.kind], what, s.mode, s.bytes, s.launches))
    return out


def gene8_pick_form(cut: bool, top_a: int, top_bt: int) -> int:
    """The auto-mode rule of gene 8 in FP64 (include/mmx.h: mmx_gene8_pick_form): 100 SA + 10 SB + levels, 0 = FP64 pipe."""
    return int(load().mmx_gene8_pick_form(int(bool(cut)), int(top_a), int(top_bt)))


def peak_probe(kind: int, device: int = 0) -> float:
    v = C.c_double()
    rc = load().mmx_peak_probe(device, kind, C.byref(v))
    if rc != OK:
        raise MmxError(rc, load().mmx_last_error(None).decode())
    return v.value


class Context:
    """Owns an mmx_ctx.  Mirrors what CudaBackend (host/include/mmx/cuda_backend.hpp) does in C++."""

    def __init__(self, n: int = 256, dtype: int = F64, numerics: int = FAST, timeout_s: float = 120.0,
                 repetitions: int = 1, num_slots: int = 1, devices=None, host_threads: int = 1,
                 launch_batching: int = 1, matmul_variant: int = 0, warmup: int = 0, pin_host: int = 1,
                 host_core_first: int = 0, host_core_count: int = 0, early_timeout: int = 1):
        self._lib = load()
        cfg = Config()
        self._lib.mmx_default_config(C.byref(cfg))
        cfg.n, cfg.dtype, cfg.numerics = n, dtype, numerics
        cfg.timeout_s, cfg.repetitions, cfg.num_slots = timeout_s, repetitions, num_slots
        cfg.host_threads, cfg.launch_batching = host_threads, launch_batching
        cfg.matmul_variant, cfg.warmup = matmul_variant, warmup
        cfg.pin_host, cfg.host_core_first, cfg.host_core_count = pin_host, host_core_first, host_core_count
        cfg.early_timeout = early_timeout
        self._devices = None
        if devices is not None:
            self._devices = (C.c_int32 * len(devices))(*devices)
            cfg.devices = C.cast(self._devices, C.POINTER(C.c_int32))
        handle = C.c_void_p()
        rc = self._lib.mmx_create(C.byref(cfg), C.byref(handle))
        if rc != OK:
            raise MmxError(rc, self._lib.mmx_last_error(None).decode())
        self._h = handle
        self.n, self.dtype = n, dtype
        self.np_dtype = np.float64 if dtype == F64 else np.float32

    def close(self):
        if getattr(self, "_h", None):
            self._lib.mmx_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != OK:
            raise MmxError(rc, self._lib.mmx_last_error(self._h).decode())

    @property
    def gene_length(self) -> int:
        return self._lib.mmx_gene_length(self._h)

    @property
    def num_slots(self) -> int:
        return self._lib.mmx_num_slots(self._h)

    def measure(self, genome, slot: int = 0) -> Outcome:
        bits = genome_bits(genome)
        out = Outcome()
        self._check(self._lib.mmx_measure(self._h, slot, bits.ctypes.data, bits.size, C.byref(out)))
        return out

    def measure_batch(self, genomes) -> list[Outcome]:
        mats = [genome_bits(g) for g in genomes]
        gene_len = mats[0].size if mats else GENE_LENGTH
        flat = np.ascontiguousarray(np.concatenate(mats)) if mats else np.zeros(0, np.uint8)
        outs = (Outcome * max(1, len(mats)))()
        self._check(self._lib.mmx_measure_batch(self._h, flat.ctypes.data, len(mats), gene_len, outs))
        return list(outs[: len(mats)])

    def stats(self, slot: int = 0) -> RunStats:
        st = RunStats()
        self._check(self._lib.mmx_last_stats(self._h, slot, C.byref(st)))
        return st

    def fetch(self, array: int, slot: int = 0) -> np.ndarray:
        out = np.empty((self.n, self.n), dtype=self.np_dtype)
        self._check(self._lib.mmx_fetch_array(self._h, slot, array, out.ctypes.data, out.nbytes))
        return out

    def fetch_rows(self, array: int, row0: int, rows: int, slot: int = 0) -> np.ndarray:
        out = np.empty((rows, self.n), dtype=self.np_dtype)
        self._check(self._lib.mmx_fetch_rows(self._h, slot, array, row0, rows, out.ctypes.data, out.nbytes))
        return out

    def upload(self, array: int, data: np.ndarray, slot: int = 0):
        data = np.ascontiguousarray(data, dtype=self.np_dtype)
        assert data.shape == (self.n, self.n)
        self._check(self._lib.mmx_upload_array(self._h, slot, array, data.ctypes.data, data.nbytes))

    def run_loop(self, gene: int, i: int = 0, j: int = 0, slot: int = 0) -> float:
        s = C.c_double(0.0)
        self._check(self._lib.mmx_run_loop(self._h, slot, gene, i, j, C.byref(s)))
        return s.value

    def run_loop_rows(self, gene: int, row0: int, rows: int, slot: int = 0) -> float:
        s = C.c_double(0.0)
        self._check(self._lib.mmx_run_loop_rows(self._h, slot, gene, row0, rows, C.byref(s)))
        return s.value

    def gene8_form(self, slot: int = 0) -> int:
        """Form the last FP64 auto-mode gene-8 launch took: 2..7 INT8 slices, 0 the FP64 pipe, -1 not applicable."""
        v = C.c_int32()
        self._check(self._lib.mmx_gene8_form(self._h, slot, C.byref(v)))
        return v.value

    def time_gene8_contraction(self, iters: int = 5, flush_l2: bool | int = True, slot: int = 0) -> float:
        """ms per launch of the gene-8 contraction alone (FP64 auto mode): operands encoded once, reused by the timed launches.
        flush_l2 = 2: the launches back to back inside one event pair (sustained rate)."""
        ms = C.c_double()
        self._check(self._lib.mmx_time_gene8_contraction(self._h, slot, iters, int(flush_l2), C.byref(ms)))
        return ms.value

    def device_ptr(self, array: int, slot: int = 0) -> int:
        p = C.c_void_p()
        self._check(self._lib.mmx_device_ptr(self._h, slot, array, C.byref(p)))
        return p.value

    # -- row-sharded run (include/mmx.h: mmx_shard_*) ---------------------------------------------
    def shard_run_local(self, slots=None) -> tuple[float, list[dict]]:
        """One individual sharded over the given slots of this context (all of them by default)."""
        slots = list(range(self.num_slots)) if slots is None else list(slots)
        arr = (C.c_int32 * len(slots))(*slots)
        stats = (ShardStats * len(slots))()
        checksum = C.c_double()
        self._check(self._lib.mmx_shard_run_local(self._h, arr, len(slots), stats, C.byref(checksum)))
        return checksum.value, [st.as_dict() for st in stats]

    def shard_export(self, slot: int = 0) -> bytes:
        h = ShardHandle()
        self._check(self._lib.mmx_shard_export(self._h, slot, C.byref(h)))
        return bytes(h)

    def shard_bind(self, rank: int, world: int, handles: list[bytes], slot: int = 0) -> None:
        table = (ShardHandle * world)()
        for r, raw in enumerate(handles):
            C.memmove(C.byref(table[r]), raw, C.sizeof(ShardHandle))
        self._check(self._lib.mmx_shard_bind(self._h, slot, rank, world, table, None))

    def shard_phase1(self, slot: int = 0) -> None:
        self._check(self._lib.mmx_shard_phase1(self._h, slot))

    def shard_phase2(self, slot: int = 0) -> dict:
        st = ShardStats()
        self._check(self._lib.mmx_shard_phase2(self._h, slot, C.byref(st)))
        return st.as_dict()

    def time_loop(self, gene: int, iters: int = 10, flush_l2: bool = True, slot: int = 0) -> float:
        ms = C.c_double()
        self._check(self._lib.mmx_time_loop(self._h, slot, gene, iters, int(flush_l2), C.byref(ms)))
        return ms.value
