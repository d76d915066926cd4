#!/bin/bash
# balanced solo launch (LG_BALANCE=1, default) vs 32-env groups (LG_BALANCE=0)
B="python bench.py --steps 20 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy"
for spec in "c5 1048576" "c5 524288" "c5 262144" "c5 131072" "c3 65536"; do
  set -- $spec
  for v in 1 0; do
    r=$(LG_BALANCE=$v $B --config $1 --envs $2 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("%.1fM kernel_ms=%.4f frac=%.3f graph_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"], d["roofline"]["frac"], d["timing"]["graph_ms_per_step"]))')
    echo "$1 envs=$2 LG_BALANCE=$v: $r"
  done
done
