#!/bin/bash
# c5 at the headline size and at the N=8 shard size for the default library and variants
for lib in default "$@"; do
  for n in 1048576 131072; do
    if [ "$lib" = default ]; then pre=""; else pre="LG_LIB_PATH=$lib"; fi
    v=$(env $pre python bench.py --envs $n --no-e2e --no-cpu-baseline --no-u8 --no-policy 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print("%.1fM kernel_ms=%.4f graph_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"], d["timing"]["graph_ms_per_step"]))' 2>&1 | tail -1)
    echo "$lib $n: $v"
  done
done
