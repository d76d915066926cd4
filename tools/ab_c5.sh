#!/bin/bash
# c5 A/B over library variants: the 2^20 batch and the 131072-env (N=8) shard
B="python bench.py --steps 20 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy --config c5"
for lib in default "$@"; do
  for n in 1048576 131072; do
    if [ "$lib" = default ]; then pre=""; else pre="LG_LIB_PATH=$lib"; fi
    r=$(env $pre $B --envs $n 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("%.1fM kernel_ms=%.4f frac=%.3f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"], d["roofline"]["frac"]))')
    echo "$lib envs=$n: $r"
  done
done
