"""TEST INFRASTRUCTURE: the unmodified reference (oracle/_ref/libacctune_ref.so, built from /root/reference by oracle/Makefile)
behind the same ctypes wrapper the product's host layer uses, so tests can drive both with identical inputs."""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

from paper_1806_01430_b200 import hostapi as H

_ref = None


def reference() -> H.Api | None:
    """The unmodified reference behind oracle/ref_shim.cpp, or None when oracle/_ref is not built."""
    global _ref
    if _ref is None:
        path = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "libacctune_ref.so"
        if not path.exists():
            return None
        _ref = H.Api(C.CDLL(str(path)), "ref")
    return _ref


def ref_probe_text(text: str, basename: str, compile_cmd: str, workdir) -> tuple[int, list[dict]]:
    """The reference's build_candidate_set with `compile_cmd` as the compiler (oracle/ref_shim.cpp: ref_probe_text)."""
    api = reference()
    buf = C.create_string_buffer(1 << 16)
    rc = api.f("probe_text")(text.encode(), basename.encode(), compile_cmd.encode(), str(workdir).encode(), buf, C.c_size_t(len(buf)))
    return rc, [json.loads(line) for line in buf.value.decode().splitlines() if line]
