#!/bin/bash
# A/B: specialised lane-team kernels vs the generic one (LG_NO_SPEC=1) on c4 and c2
B="python bench.py --steps 20 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy"
for c in ${@:-c4 c2}; do
  for v in 0 1; do
    r=$(LG_NO_SPEC=$v $B --config $c 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("%.1fM kernel_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"]))')
    echo "$c LG_NO_SPEC=$v: $r"
  done
done
