# rate probes of the contraction kernel (results are wrong under MMX_OZ_DEBUG != 0): bash tools/oz_debug_probe.sh "<debug values>" "<sizes>"
for d in ${1:-0 1 2 3}; do echo "MMX_OZ_DEBUG=$d"; MMX_OZ_DEBUG=$d python tools/gene8_auto_time.py ${2:-4096 8192} 2>&1 | cut -c1-330; done
