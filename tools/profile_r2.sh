#!/bin/bash
# r2 ncu captures of the team / solo step kernels (c4, c2, c3) and the 131k-env c5 shard
#   bash tools/profile_r2.sh <tag> [configs...]
tag=${1:-r2}; shift
cfgs=${@:-c4 c2 c3}
B="python bench.py --steps 2 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy --no-graph"
for c in $cfgs; do
  case $c in
    c4|c2) k=regex:env_kernel ;;
    c3) k=regex:env_solo_kernel_dungeon ;;
    c5s|c5) k=regex:env_solo_kernel_binary ;;
  esac
  extra=""; cc=$c
  if [ $c = c5s ]; then extra="--envs 131072"; cc=c5; fi
  $B --config $cc $extra > gpurun_out/plain_$c.log 2>&1 || { echo "plain $c failed"; tail -5 gpurun_out/plain_$c.log; continue; }
  timeout 600 ncu --set full --clock-control none --import-source on -k $k -s 3 -c 1 -o gpurun_out/${tag}_full_$c -f $B --config $cc $extra > gpurun_out/ncu_$c.log 2>&1
  tail -1 gpurun_out/ncu_$c.log
done
# digest on the box (the reports are too large to travel back together)
for c in $cfgs; do
  rep=gpurun_out/${tag}_full_$c.ncu-rep
  [ -f $rep ] || continue
  python profiles/ncu_summary.py $rep 40 > gpurun_out/${tag}_ncu_$c.txt 2>&1
  ncu -i $rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src_$c.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/${tag}_src_$c.csv 60 > gpurun_out/${tag}_lines_$c.txt 2>&1
  rm -f gpurun_out/${tag}_src_$c.csv
  [ "$KEEP_REP" = 1 ] || rm -f $rep
done
