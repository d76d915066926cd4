#!/bin/bash
# Launch-policy sweep (env overrides of the host's kernel choice); one JSON field per line.
B="python bench.py --no-e2e --no-cpu-baseline --no-u8"
run() { # name env... -- config
  local name=$1; shift
  local v=$(env "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print("%.1fM kernel_ms=%.4f frac=%.3f" % (d["value"]/1e6, d["roofline"]["step_kernel_ms"], d["roofline"]["frac"]))' 2>&1 | tail -1)
  echo "$name: $v"
}
run "c3 default" $B --config c3
run "c3 team" LG_FORCE_TEAM=1 $B --config c3
run "c3 solo32" LG_SOLO_THREADS=32 $B --config c3
run "c3 solo128" LG_SOLO_THREADS=128 $B --config c3
run "c3 slot" LG_STREAM=0 $B --config c3
run "c2 default" $B --config c2
run "c2 solo" LG_SOLO_MID=1 $B --config c2
run "c2 team32thr" LG_TEAM_THREADS=32 $B --config c2
run "c2 team128thr" LG_TEAM_THREADS=128 $B --config c2
run "c1 default" $B --config c1
run "c1 team" LG_FORCE_TEAM=1 $B --config c1
run "c4 default" $B --config c4
run "c4 team32thr" LG_TEAM_THREADS=32 $B --config c4
run "c4 team128thr" LG_TEAM_THREADS=128 $B --config c4
run "c5 solo32" LG_SOLO_THREADS=32 $B --config c5
run "c5 solo128" LG_SOLO_THREADS=128 $B --config c5
