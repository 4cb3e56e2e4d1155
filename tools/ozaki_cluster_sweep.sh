#!/bin/bash
# FP64-on-INT8 contraction: stage width (MMX_OZ_BK) and cluster size (multicast of the a slices, MMX_OZ_CLUSTER)
# against kernel time and accuracy.  usage: ozaki_cluster_sweep.sh "bk:cluster" ...
for cfg in ${@:-32:1 64:1 32:2 64:4}; do bk=${cfg%%:*}; c=${cfg##*:}; echo "== MMX_OZ_BK=$bk MMX_OZ_CLUSTER=$c"
  MMX_OZ_BK=$bk MMX_OZ_CLUSTER=$c timeout 300 python tools/ozaki_probe.py 300 4096 8192 2>&1 | grep '"variant": 40,' | tail -3; done
