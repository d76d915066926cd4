#!/bin/bash
# ncu evidence for profiles/ (run under gpurun on one B200):
#   bash tools/profile_round.sh <tag>
# 1. plain bench runs (must exit 0 before ncu touches them)
# 2. launch list of the c5 bench (device time + DRAM bytes per launch)
# 3. one `--set full` capture of the step kernel for c5, c3 and c4
set -e
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-u8"
for c in c5 c3 c4; do
  $B --config $c > $out/plain_$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $out/${tag}_launches_c5.csv $B --config c5 > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:env_solo_kernel_binary -s 3 -c 1 \
    -o $out/${tag}_full_c5 -f $B --config c5 > $out/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:env_solo_kernel_dungeon -s 3 -c 1 \
    -o $out/${tag}_full_c3 -f $B --config c3 > $out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:env_kernel -s 3 -c 1 \
    -o $out/${tag}_full_c4 -f $B --config c4 > $out/ncu_c4.log 2>&1
echo profile done
