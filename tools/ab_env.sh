#!/bin/bash
# generic A/B: CONFIG ENVS then env-var assignments per variant, e.g.
#   bash tools/ab_env.sh c3 65536 "" "LG_FORCE_TEAM=1" "LG_EARLY=1"
c=$1; n=$2; shift 2
B="python bench.py --steps 20 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy"
for v in "$@"; do
  r=$(env $v $B --config $c --envs $n 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("%.1fM kernel_ms=%.4f frac=%.3f graph_ms=%.4f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"], d["roofline"]["frac"], d["timing"]["graph_ms_per_step"]))')
  echo "$c envs=$n [$v]: $r"
done
