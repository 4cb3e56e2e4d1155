"""ctypes binding of host/include/mmxhost/capi_host.h (the C window onto the C++ host layer).

`Api` takes a library and a symbol prefix, so the tests can point the same wrapper at the unmodified reference
behind oracle/ref_shim.cpp (same function shapes with a `ref_` prefix; the loader for that lives in tests/refapi.py --
nothing in this package opens anything under oracle/).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "lib"
STATUS_NAMES = ("measured", "compile_error", "runtime_error", "timeout")

E_ERROR, E_LENGTH, E_TOOLCHAIN, E_WORKDIR, E_ZERO_FITNESS, E_UNAVAILABLE, E_NONPOSITIVE, E_CONFIG, E_NOCANDIDATES, E_MODEL = range(-1, -11, -1)


class Outcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("time_s", C.c_double), ("wall_cost_s", C.c_double)]

    def as_tuple(self):
        return (self.status, self.time_s, self.wall_cost_s)


class GAParams(C.Structure):
    _fields_ = [("population", C.c_int32), ("generations", C.c_int32), ("crossover_rate", C.c_double),
                ("mutation_rate", C.c_double), ("seed", C.c_uint64), ("elite_count", C.c_int32)]


class CudaConfig(C.Structure):
    _fields_ = [("n", C.c_int32), ("dtype", C.c_int32), ("numerics", C.c_int32), ("timeout_s", C.c_double),
                ("repetitions", C.c_int32), ("warmup", C.c_int32), ("host_threads", C.c_int32),
                ("launch_batching", C.c_int32), ("matmul_variant", C.c_int32), ("num_devices", C.c_int32),
                ("devices", C.POINTER(C.c_int32))]


MEASURE_CB = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint8), C.c_size_t, C.POINTER(Outcome), C.c_void_p)


class HostError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"host error {code}: {message}")
        self.code = code


def _bits(genome) -> np.ndarray:
    if isinstance(genome, str):
        return np.frombuffer(genome.encode(), dtype=np.uint8) - ord("0")
    return np.ascontiguousarray(np.asarray(genome, dtype=np.uint8))


def _str(arr) -> str:
    return "".join("1" if x else "0" for x in arr)


class Api:
    """One of the two implementations: prefix 'mmxh' (this repo) or 'ref' (the reference)."""

    def __init__(self, lib: C.CDLL, prefix: str):
        self.lib, self.prefix = lib, prefix
        self.f("last_error").restype = C.c_char_p
        self.f("status_name").restype = C.c_char_p
        for name in ("evaluator_create_cb", "evaluator_create_sim", "evaluator_create_cuda"):
            if hasattr(lib, f"{prefix}_{name}"):
                self.f(name).restype = C.c_void_p

    def f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def check(self, rc):
        if rc < 0:
            raise HostError(rc, self.f("last_error")().decode())
        return rc

    # ---- GA pieces ---------------------------------------------------------------------------
    def rng_draws(self, seed, kind, count, n_arg=0):
        vals, raws = (C.c_double * count)(), (C.c_uint64 * count)()
        self.check(self.f("rng_draws")(C.c_uint64(seed), kind, C.c_uint64(n_arg), C.c_size_t(count), vals, raws))
        return [int(x) for x in raws] if kind == 3 else list(vals)

    def fitness_from_time(self, t):
        f = C.c_double()
        self.check(self.f("fitness_from_time")(C.c_double(t), C.byref(f)))
        return f.value

    def assign_fitness(self, status, times):
        m = len(status)
        out = (C.c_double * m)()
        self.check(self.f("assign_fitness")((C.c_int32 * m)(*status), (C.c_double * m)(*times), C.c_size_t(m), out))
        return list(out)

    def init_population(self, a, m, seed):
        bits = (C.c_uint8 * (a * m))()
        self.check(self.f("init_population")(C.c_size_t(a), m, C.c_uint64(seed), bits))
        return [_str(bits[i * a:(i + 1) * a]) for i in range(m)]

    def breed(self, genomes, fitness, pc, pm, elite, seed, skip=0):
        m, a = len(genomes), len(genomes[0])
        flat = (C.c_uint8 * (a * m))(*[int(ch) for g in genomes for ch in g])
        nxt = (C.c_uint8 * (a * m))()
        self.check(self.f("breed")(flat, (C.c_double * m)(*fitness), C.c_size_t(m), C.c_size_t(a), C.c_double(pc),
                                   C.c_double(pm), elite, C.c_uint64(seed), C.c_uint64(skip), nxt))
        return [_str(nxt[i * a:(i + 1) * a]) for i in range(m)]

    def roulette(self, fitness, count, seed):
        m = len(fitness)
        picks = (C.c_int32 * count)()
        self.check(self.f("roulette")((C.c_double * m)(*fitness), C.c_size_t(m), C.c_size_t(count), C.c_uint64(seed), picks))
        return list(picks)

    def mutate(self, genome, pm, seed):
        a = len(genome)
        out = (C.c_uint8 * a)()
        self.check(self.f("mutate")((C.c_uint8 * a)(*[int(c) for c in genome]), C.c_size_t(a), C.c_double(pm), C.c_uint64(seed), out))
        return _str(out)

    def one_point_crossover(self, p1, p2, seed):
        a = len(p1)
        c1, c2 = (C.c_uint8 * a)(), (C.c_uint8 * a)()
        self.check(self.f("one_point_crossover")((C.c_uint8 * a)(*[int(c) for c in p1]), (C.c_uint8 * a)(*[int(c) for c in p2]),
                                                 C.c_size_t(a), C.c_uint64(seed), c1, c2))
        return _str(c1), _str(c2)

    # ---- sim model -----------------------------------------------------------------------------
    def model_time_all(self, model_path, a):
        times = np.zeros(1 << a, dtype=np.float64)
        rc = self.check(self.f("model_time_all")(str(model_path).encode(), times.ctypes.data_as(C.POINTER(C.c_double)), C.c_size_t(times.size)))
        assert rc == a
        return times

    def exhaustive_best(self, model_path, a):
        bits, t = (C.c_uint8 * a)(), C.c_double()
        self.check(self.f("exhaustive_best")(str(model_path).encode(), bits, C.c_size_t(a), C.byref(t)))
        return _str(bits), t.value

    def status_name(self, status):
        return self.f("status_name")(status).decode()


class Evaluator:
    """Handle on an Evaluator of either implementation."""

    def __init__(self, api: Api, handle, keep=None):
        if not handle:
            raise HostError(-1, api.f("last_error")().decode())
        self.api, self.h, self._keep = api, C.c_void_p(handle), keep

    @classmethod
    def from_callback(cls, api: Api, genes: int, fn, jobs: int = 1, cache_file=None):
        """fn(genome_str) -> (status, time_s, wall_cost_s) | raises ToolchainMissingSignal/Exception"""
        def trampoline(bits, n, out, _user):
            try:
                res = fn(_str(bits[:n]))
            except ToolchainMissingSignal:
                return -3
            except Exception:
                return -1
            out.contents.status, out.contents.time_s, out.contents.wall_cost_s = res
            return 0
        cb = MEASURE_CB(trampoline)
        h = api.f("evaluator_create_cb")(C.c_size_t(genes), cb, None, jobs, str(cache_file).encode() if cache_file else None)
        return cls(api, h, keep=cb)

    @classmethod
    def from_sim(cls, api: Api, model_path, jobs: int = 1, cache_file=None):
        h = api.f("evaluator_create_sim")(str(model_path).encode(), jobs, str(cache_file).encode() if cache_file else None)
        return cls(api, h)

    @classmethod
    def from_cuda(cls, api: Api, n=256, dtype=0, numerics=0, timeout_s=120.0, repetitions=1, warmup=0, host_threads=1,
                  launch_batching=1, matmul_variant=0, devices=(0,), cache_file=None):
        devs = (C.c_int32 * len(devices))(*devices)
        cfg = CudaConfig(n, dtype, numerics, timeout_s, repetitions, warmup, host_threads, launch_batching, matmul_variant,
                         len(devices), C.cast(devs, C.POINTER(C.c_int32)))
        h = api.f("evaluator_create_cuda")(C.byref(cfg), str(cache_file).encode() if cache_file else None)
        if not h:
            msg = api.f("last_error")().decode()
            code, _, text = msg.partition(":")
            raise HostError(int(code) if code.lstrip("-").isdigit() else -1, text or msg)
        return cls(api, h, keep=devs)

    def close(self):
        if self.h:
            self.api.f("evaluator_destroy")(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def evaluate(self, genome):
        bits = _bits(genome)
        out = Outcome()
        self.api.check(self.api.f("evaluator_evaluate")(self.h, bits.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_size_t(bits.size), C.byref(out)))
        return out.as_tuple()

    def evaluate_all(self, genomes):
        if not genomes:
            return []
        n = len(genomes[0])
        flat = np.ascontiguousarray(np.concatenate([_bits(g) for g in genomes]))
        outs = (Outcome * len(genomes))()
        self.api.check(self.api.f("evaluator_evaluate_all")(self.h, flat.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_size_t(len(genomes)), C.c_size_t(n), outs))
        return [o.as_tuple() for o in outs]

    def set_costs(self, genomes, costs):
        """Longest-first scheduling of evaluate_all (mmxhost only): genomes with a larger predicted cost start first."""
        n = len(genomes[0])
        flat = np.ascontiguousarray(np.concatenate([_bits(g) for g in genomes]))
        arr = np.ascontiguousarray(costs, dtype=np.float64)
        assert arr.size == len(genomes)
        self.api.check(self.api.f("evaluator_set_costs")(self.h, flat.ctypes.data_as(C.POINTER(C.c_uint8)),
                                                         arr.ctypes.data_as(C.POINTER(C.c_double)), C.c_size_t(len(genomes)), C.c_size_t(n)))

    def counters(self):
        c4, el = (C.c_uint64 * 4)(), C.c_double()
        self.api.check(self.api.f("evaluator_counters")(self.h, c4, C.byref(el)))
        return {"requests": c4[0], "distinct": c4[1], "cache_hits": c4[2], "backend_calls": c4[3], "elapsed_s": el.value}

    def run_ga(self, population=12, generations=12, crossover_rate=0.9, mutation_rate=0.05, seed=1, elite_count=1, genes=12):
        """Only for the mmxh implementation (the reference shim has its own run_ga entry points)."""
        p = GAParams(population, generations, crossover_rate, mutation_rate, seed, elite_count)
        csv = C.create_string_buffer(1 << 16)
        best = (C.c_uint8 * 64)()
        best_s, base_s = C.c_double(), C.c_double()
        n = self.api.check(self.api.f("run_ga")(self.h, C.byref(p), csv, C.c_size_t(1 << 16), best, C.byref(best_s), C.byref(base_s)))
        assert n < (1 << 16)
        return {"csv": csv.value.decode(), "best_genome": _str(best[:genes]), "best_s": best_s.value, "baseline_s": base_s.value}


def predicted_cost(genome, n=256, dtype=0, numerics=0, timeout_s=120.0, repetitions=1, warmup=0, host_threads=1) -> float:
    """The static estimate MultiGpuEvaluator orders a batch by (seconds, order of magnitude; 0 for infeasible genomes)."""
    api = mine()
    fn = api.lib.mmxh_predicted_cost
    fn.restype = C.c_double
    cfg = CudaConfig(n, dtype, numerics, timeout_s, repetitions, warmup, host_threads, 1, 0, 0, None)
    bits = _bits(genome)
    return float(fn(C.byref(cfg), bits.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_size_t(bits.size)))


class ToolchainMissingSignal(Exception):
    """Raise from a callback backend to make the C++ side throw ToolchainMissing."""


_mine = None

def mine() -> Api:
    global _mine
    if _mine is None:
        path = LIB_DIR / "libmmx_host.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} is missing: run `python -m paper_1806_01430_b200.build`")
        _mine = Api(C.CDLL(str(path)), "mmxh")
    return _mine


def dump_number(v: float) -> str:
    buf = C.create_string_buffer(64)
    mine().lib.mmxh_dump_number(C.c_double(v), buf, C.c_size_t(64))
    return buf.value.decode()


# ---- source model and commands (source_model.hpp, commands.hpp) -------------------------------------

def scan_loops(api: Api, text: str, label: str = "<text>") -> list[dict]:
    """scan_loops on in-memory text: id, line, depth, header_start, body_begin, body_end, indent_len per loop."""
    rows = (C.c_int64 * (7 * 256))()
    n = api.check(api.f("scan_loops")(label.encode(), text.encode(), rows, C.c_size_t(256)))
    keys = ("id", "line", "depth", "header_start", "body_begin", "body_end", "indent_len")
    return [dict(zip(keys, (int(rows[7 * k + q]) for q in range(7)))) for k in range(n)]


def render_variant(api: Api, text: str, genome) -> str:
    bits = _bits(genome)
    buf = C.create_string_buffer(len(text.encode()) + 64 * (bits.size + 1) + 64)
    api.check(api.f("render_variant")(text.encode(), bits.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_size_t(bits.size), buf, C.c_size_t(len(buf))))
    return buf.value.decode()


def strip_directives(api: Api, text: str) -> str:
    buf = C.create_string_buffer(len(text.encode()) + 16)
    api.check(api.f("strip_directives")(text.encode(), buf, C.c_size_t(len(buf))))
    return buf.value.decode()


def _run_command(fn, *args) -> tuple[int, str, str]:
    out, err = C.create_string_buffer(1 << 16), C.create_string_buffer(1 << 16)
    rc = fn(*args, out, C.c_size_t(len(out)), err, C.c_size_t(len(err)))
    return rc, out.value.decode(), err.value.decode()


def cmd_tune(api: Api, config_path, seed=None, sim_model=None) -> tuple[int, str, str]:
    """(exit code, stdout, stderr) of `tune <config> [--seed N] [--sim model]`."""
    return _run_command(api.f("cmd_tune"), str(config_path).encode(), int(seed is not None), C.c_uint64(seed or 0),
                        str(sim_model).encode() if sim_model else None)


def cmd_report(api: Api, workdir) -> tuple[int, str, str]:
    return _run_command(api.f("cmd_report"), str(workdir).encode())


def cmd_analyze(api: Api, config_path) -> tuple[int, str, str]:
    return _run_command(api.f("cmd_analyze"), str(config_path).encode())


# ---- static feasibility and kernel matching (feasibility.hpp, kernel_match.hpp) ----------------------------

def probe_source(text: str, label: str = "<text>") -> tuple[int, list[dict]]:
    """(accepted loop count or negative error class, probe report rows) of this repo's static probe."""
    import json
    api = mine()
    buf = C.create_string_buffer(1 << 16)
    rc = api.f("probe_source")(label.encode(), text.encode(), buf, C.c_size_t(len(buf)))
    return rc, [json.loads(line) for line in buf.value.decode().splitlines() if line]


def variant_feasible(text: str, genome, label: str = "<text>") -> tuple[bool, list[str]]:
    api = mine()
    bits = _bits(genome)
    buf = C.create_string_buffer(1 << 14)
    rc = api.check(api.f("variant_feasible")(label.encode(), text.encode(), bits.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_size_t(bits.size),
                                             buf, C.c_size_t(len(buf))))
    return rc == 1, buf.value.decode().splitlines()


def match_kernels(text: str, label: str = "<text>") -> dict:
    import json
    api = mine()
    buf = C.create_string_buffer(1 << 16)
    api.check(api.f("match_kernels")(label.encode(), text.encode(), buf, C.c_size_t(len(buf))))
    return json.loads(buf.value.decode())


# ---- calibration (calibrate.hpp) ------------------------------------------------------------------------------

def calibrate(genomes, times, n: int, dtype: int = 0) -> dict:
    """Fit the plan model to measured (genome, seconds) samples and project it onto the reference's cost-model JSON."""
    api = mine()
    flat = np.ascontiguousarray(np.concatenate([_bits(g) for g in genomes]).astype(np.uint8))
    t = np.ascontiguousarray(np.asarray(times, dtype=np.float64))
    buf = C.create_string_buffer(1 << 18)
    plan, rep, best = np.zeros(22), np.zeros(8), np.zeros(24, dtype=np.uint8)
    api.check(api.f("calibrate")(flat.ctypes.data_as(C.POINTER(C.c_uint8)), t.ctypes.data_as(C.POINTER(C.c_double)), C.c_size_t(len(genomes)),
                                 n, dtype, buf, C.c_size_t(len(buf)), plan.ctypes.data_as(C.POINTER(C.c_double)),
                                 rep.ctypes.data_as(C.POINTER(C.c_double)), best.ctypes.data_as(C.POINTER(C.c_uint8))))
    keys = ("fit_rms_rel_err", "fit_max_rel_err", "projection_rms_rel_err", "projection_max_rel_err", "plan_best_s", "cost_best_s",
            "inexact_loops", "samples")
    return {"model_json": buf.value.decode(), "plan": plan, "report": dict(zip(keys, map(float, rep))),
            "plan_best": _str(best[:12]), "cost_best": _str(best[12:])}


def plan_model_times(plan22, n: int, dtype: int = 0) -> np.ndarray:
    """Seconds of all 4096 genomes under a plan model (index = sum bit_k << k); -1 for infeasible genomes."""
    api = mine()
    p = np.ascontiguousarray(np.asarray(plan22, dtype=np.float64))
    out = np.zeros(4096)
    api.check(api.f("plan_model_times")(p.ctypes.data_as(C.POINTER(C.c_double)), n, dtype, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def cmd_calibrate(api: Api, config_path) -> tuple[int, str, str]:
    return _run_command(api.f("cmd_calibrate"), str(config_path).encode())
