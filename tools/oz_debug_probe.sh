for d in ${@:-0 1 2 3}; do echo "MMX_OZ_DEBUG=$d"; MMX_OZ_DEBUG=$d python tools/gene8_auto_time.py 4096 8192 2>&1 | cut -c1-330; done
