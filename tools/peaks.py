#!/usr/bin/env python
"""Measures the roofline denominators MEASURED_PEAKS.json lacks (FP64 DFMA / DMMA, FP32 FFMA) and
this library's own HBM copy / write / read rates; writes one JSON object (stdout or --out)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1806_01430_b200 import capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    args = ap.parse_args()
    res = {
        "hbm_copy_gbs": capi.peak_probe(capi.PEAK_COPY),
        "hbm_write_gbs": capi.peak_probe(capi.PEAK_WRITE),
        "hbm_read_gbs": capi.peak_probe(capi.PEAK_READ),
        "fp64_fma_tflops": capi.peak_probe(capi.PEAK_FP64_FMA),
        "fp64_dmma_tflops": capi.peak_probe(capi.PEAK_FP64_DMMA),
        "fp32_fma_tflops": capi.peak_probe(capi.PEAK_FP32_FMA),
        "umma_i8_tops": capi.peak_probe(capi.PEAK_UMMA_I8),
        "umma_tf32_tflops": capi.peak_probe(capi.PEAK_UMMA_TF32),
        "umma_bf16_tflops": capi.peak_probe(capi.PEAK_UMMA_BF16),
        "how": "csrc/peaks.cu: best of N CUDA-event-timed launches after 3 warm-ups; 16 independent FMA/DMMA chains "
               "per thread, 4 CTAs x 256 threads per SM; HBM probes move 2 GiB buffers with 128-bit accesses; umma_*: tcgen05.mma "
               "M=128 x N=256 instructions back to back on operands resident in shared memory, one issuing thread per SM (issue peak of the tensor pipe)",
    }
    text = json.dumps(res, indent=1)
    print(text)
    if args.out:
        Path(args.out).write_text(text + "\n")


if __name__ == "__main__":
    main()
