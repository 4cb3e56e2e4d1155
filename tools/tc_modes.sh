#!/bin/bash
# accuracy (error over the 1e-6 norm-wise bar) and speed of the FP32 tensor-core contraction per MMX_TC_MODE
for m in ${@:-14802 14803 14804 14816 13804}; do echo "== mode $m"; MMX_TC_MODE=$m timeout 300 python tools/tc_probe.py 1000 4096 8192 2>&1 | tail -9; done
