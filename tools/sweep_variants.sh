#!/bin/bash
# A/B of prebuilt library variants (variants/*.so) on given configs: bash tools/sweep_variants.sh "c4 c2" variants/a.so ...
cfgs=$1; shift
for lib in default "$@"; do
  for c in $cfgs; do
    if [ "$lib" = default ]; then pre=""; else pre="LG_LIB_PATH=$lib"; fi
    v=$(env $pre python bench.py --config $c --no-e2e --no-cpu-baseline --no-u8 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print("%.1fM kernel_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"]))' 2>&1 | tail -1)
    echo "$lib $c: $v"
  done
done
