#!/bin/bash
B="python bench.py --no-e2e --no-cpu-baseline --no-u8 --no-policy"
for args in "--config c5" "--config c3" "--config c5 --envs 131072" "--config c5 --envs 262144"; do
  for ne in 0 1; do
    if [ $ne = 1 ]; then pre="LG_NO_EARLY=1"; else pre=""; fi
    v=$(env $pre $B $args 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print("%.1fM kernel_ms=%.4f eager_ms=%.4f graph_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"], d["timing"]["eager_ms_per_step"], d["timing"]["graph_ms_per_step"]))' 2>&1 | tail -1)
    echo "$args no_early=$ne: $v"
  done
done
