"""C ABI checks that need no GPU: the library loads, exports every symbol include/mmx.h
declares, the catalogue and planner agree with the reference-generated golden vectors, and the
product refuses to run without a CUDA device (no CPU fallback)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1806_01430_b200 import capi

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "mmx.h").read_text()
    return sorted(set(re.findall(r"MMX_API\s+[\w\s\*]+?\b(mmx_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    names = header_symbols()
    assert len(names) >= 16
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/mmx.h but not exported"
    assert set(names) == set(capi._SIGNATURES), "capi.py binding table is out of sync with mmx.h"


def test_struct_sizes_match_header_layout():
    import ctypes as C
    cfg = capi.Config()
    capi.load().mmx_default_config(C.byref(cfg))
    assert cfg.struct_size == C.sizeof(capi.Config)
    assert (cfg.n, cfg.dtype, cfg.repetitions, cfg.timeout_s) == (256, capi.F64, 1, 120.0)


def test_catalogue_matches_reference_scan(golden):
    # golden: scan_loops() of the reference over fixtures/matmul.c
    ref = golden("catalogue.json")
    mine = capi.loop_catalogue()
    assert len(mine) == len(ref) == capi.GENE_LENGTH
    for r, m in zip(ref, mine):
        assert (m["gene"], m["line"], m["depth"]) == (r["id"], r["line"], r["depth"])


def all_genomes():
    for mask in range(1 << 12):
        yield mask, "".join("1" if (mask >> k) & 1 else "0" for k in range(12))


def test_feasibility_matches_mockacc_for_all_4096_genomes(golden):
    verdict = golden("feasibility_mockacc.txt").strip()
    assert len(verdict) == 4096 and verdict.count("1") == 648
    for mask, g in all_genomes():
        assert capi.plan(g, 256).feasible == int(verdict[mask]), g


def test_plan_lower_bound_met_for_every_feasible_genome():
    for n, dtype, esz in ((256, capi.F64, 8), (96, capi.F32, 4)):
        for mask, g in all_genomes():
            p = capi.plan(g, n, dtype)
            if not p.feasible:
                assert p.num_steps == 0 and p.conflict_nest >= 0
                continue
            assert (p.h2d_bytes, p.d2h_bytes) == (p.h2d_lower_bound, p.d2h_lower_bound), g
            assert p.h2d_bytes % (n * esz) == 0


def test_plan_known_answers():
    n, mb = 8192, 8192 * 8192 * 8
    p = capi.plan("101010101001", n)          # six nests on the GPU
    assert (p.h2d_bytes, p.d2h_bytes, p.kernel_launches) == (0, 8, 6)
    assert [s[0] for s in capi.plan_steps(p)] == ["gpu"] * 6 + ["d2h_sum"]
    p = capi.plan("001010101001", n)          # init-a on the CPU => a crosses once
    assert (p.h2d_bytes, p.d2h_bytes) == (mb, 8)
    p = capi.plan("101010001001", n)          # transpose on the CPU => b down, bt up
    assert (p.h2d_bytes, p.d2h_bytes) == (mb, mb + 8)
    p = capi.plan("101010101000", n)          # trace on the CPU => only the diagonal of c
    assert (p.h2d_bytes, p.d2h_bytes) == (0, n * 8)
    assert capi.plan_steps(p)[-2][0] == "d2h_diag"
    p = capi.plan("000000001001", n)          # only matmul + trace on the GPU
    assert (p.h2d_bytes, p.d2h_bytes) == (3 * mb, 8)
    p = capi.plan("101010100001", n)          # matmul on the CPU, trace on the GPU
    assert (p.h2d_bytes, p.d2h_bytes) == (n * 8, 3 * mb + 8)
    p = capi.plan("000000000000", n)          # the baseline never touches the device
    assert (p.h2d_bytes, p.d2h_bytes, p.kernel_launches) == (0, 0, 0)
    assert all(s[0] == "cpu" for s in capi.plan_steps(p))
    p = capi.plan("010000000000", 256)        # inner loop of init-a: N launches, a comes back for the CPU matmul
    assert p.kernel_launches == 256 and p.d2h_bytes == 256 * 256 * 8 and p.modes[0] == capi.MODE_GPU_INNER
    p = capi.plan("000000000010", 256)        # k loop of the matmul: N^2 launches
    assert p.kernel_launches == 256 * 256 and p.modes[4] == capi.MODE_GPU_INNER2


def test_plan_rejects_bad_arguments():
    with pytest.raises(capi.MmxError) as e:
        capi.plan("1010", 256)
    assert e.value.code == capi.E_LENGTH       # GenomeLengthMismatch analogue
    with pytest.raises(capi.MmxError) as e:
        capi.plan("0" * 12, 0)
    assert e.value.code == capi.E_INVALID


def test_no_device_means_no_context():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(capi.MmxError) as e:
        capi.Context(n=64)
    assert e.value.code == capi.E_NODEVICE     # ToolchainMissing analogue: there is no CPU fallback
    with pytest.raises(capi.MmxError):
        capi.peak_probe(capi.PEAK_COPY)


def test_genome_bits_helper():
    assert list(capi.genome_bits("101000011000")) == [1, 0, 1, 0, 0, 0, 0, 1, 1, 0, 0, 0]
    with pytest.raises(ValueError):
        capi.genome_bits("10x")
    assert capi.genome_bits(np.array([1, 0, 1])).dtype == np.uint8
