"""Builds the native libraries in-tree (they travel to the GPU box with the snapshot).

  lib/libmmx.so       CUDA kernels (sm_100a) + executor + the C ABI of include/mmx.h
  lib/libmmx_host.so  C++ host mirror of the reference tuner API (Genome, Evaluator, GA, ...)
  bin/mmx_tune        analyze | tune | report command line over the same host layer

nvcc cross-compiles without a GPU.  Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
LIB = PKG / "lib"
BIN = PKG / "bin"
OBJ = PKG / "build"

NVCC = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CXX = os.environ.get("CXX") or shutil.which("g++") or "g++"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-O2", f"-I{ROOT / 'include'}", f"-I{CSRC}",
]
# host loops are the CPU side of a genome: same arithmetic as `gcc -O2` on baseline x86-64
# (no FMA contraction), see csrc/host_loops.hpp
CXX_FLAGS = ["-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wextra",
             f"-I{ROOT / 'include'}", f"-I{CSRC}"]
HOST_CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wextra",
                  f"-I{ROOT / 'include'}", f"-I{HOST / 'include'}"]


def _newest(paths) -> float:
    return max((p.stat().st_mtime for p in paths if p.exists()), default=0.0)


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("build step failed:\n  " + " ".join(map(str, cmd)) + "\n" + proc.stdout + proc.stderr)


def _compile(src: Path, obj: Path, headers_mtime: float, verbose: bool) -> bool:
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, headers_mtime):
        return False
    if src.suffix == ".cu":
        cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    elif src.parent == CSRC:
        cmd = [CXX, *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [CXX, *HOST_CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(map(str, cmd)), flush=True)
    _run(cmd)
    return True


def build_libmmx(verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    OBJ.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [ROOT / "include" / "mmx.h", Path(__file__)]
    hm = _newest(headers)
    objs = [OBJ / (s.name + ".o") for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        changed = list(ex.map(lambda so: _compile(so[0], so[1], hm, verbose), zip(srcs, objs)))
    out = LIB / "libmmx.so"
    if any(changed) or not out.exists():
        # this image's g++ links libstdc++ statically: keep those symbols private so they cannot
        # interpose with the libstdc++.so.6 that torch / numpy load into the same process
        _run([NVCC, "-shared", "-o", str(out), *map(str, objs), "-cudart", "static", "-Xlinker", "-Bsymbolic",
              "-Xlinker", "--exclude-libs,ALL", "-lpthread", "-ldl", "-lrt"])
    return out


def build_libmmx_host(verbose: bool = False) -> Path | None:
    srcs = sorted((HOST / "src").glob("*.cpp"))
    if not srcs:
        return None
    LIB.mkdir(exist_ok=True)
    OBJ.mkdir(exist_ok=True)
    headers = list((HOST / "include").rglob("*.hpp")) + [ROOT / "include" / "mmx.h", Path(__file__)]
    hm = _newest(headers)
    objs = [OBJ / ("host_" + s.name + ".o") for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        changed = list(ex.map(lambda so: _compile(so[0], so[1], hm, verbose), zip(srcs, objs)))
    out = LIB / "libmmx_host.so"
    if any(changed) or not out.exists():
        # libmmx.so is resolved at run time next to this library
        _run([CXX, "-shared", "-o", str(out), *map(str, objs), f"-L{LIB}", "-lmmx", "-Wl,-rpath,$ORIGIN", "-Wl,-Bsymbolic",
              "-Wl,--exclude-libs,ALL", "-lpthread"])
    # the command-line front end (analyze | tune | report): the same objects, linked into an executable
    cli_src = HOST / "tools" / "mmx_tune.cpp"
    if cli_src.exists():
        BIN.mkdir(exist_ok=True)
        cli_obj = OBJ / "host_cli_mmx_tune.o"
        cli_changed = _compile(cli_src, cli_obj, hm, verbose)
        exe = BIN / "mmx_tune"
        if any(changed) or cli_changed or not exe.exists():
            core = [o for o in objs if "capi_host" not in o.name]
            _run([CXX, "-o", str(exe), str(cli_obj), *map(str, core), f"-L{LIB}", "-lmmx", "-Wl,-rpath,$ORIGIN/../lib", "-lpthread"])
    return out


def build_oracle(verbose: bool = False) -> None:
    """The CPU checker (test infrastructure).  `make ref` only where /root/reference exists."""
    targets = ["oracle"]
    if Path("/root/reference/proj/src").is_dir():
        targets.append("ref")
    cmd = ["make", "-C", str(ROOT / "oracle"), "-j8", *targets]
    if verbose:
        print(" ".join(cmd), flush=True)
    _run(cmd)


def build_all(verbose: bool = False) -> None:
    build_libmmx(verbose)
    build_libmmx_host(verbose)
    build_oracle(verbose)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print("built:", *(p.name for p in LIB.glob("*.so")))
