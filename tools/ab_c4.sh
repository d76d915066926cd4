#!/bin/bash
# c4 A/B: library variants (LG_LIB_PATH) x LG_EARLY
B="python bench.py --steps 20 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy --config ${CFG:-c4}"
for lib in default "$@"; do
  for e in 1 0; do
    if [ "$lib" = default ]; then pre=""; else pre="LG_LIB_PATH=$lib"; fi
    r=$(env $pre LG_EARLY=$e $B 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("%.1fM kernel_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"]))')
    echo "$lib early=$e: $r"
  done
done
