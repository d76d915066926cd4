#!/bin/bash
# end-of-session ncu captures (two per call: gpurun brings back <= 64 MiB):
#   bash tools/profile_final.sh "c3 conv1"   |   bash tools/profile_final.sh "c2 c4"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-graph"
for what in $1; do
  case $what in
    conv1) python tools/conv1_time.py 16384 > gpurun_out/plain_conv1.log 2>&1 || exit 1
           ncu --set full --clock-control none --import-source on -k regex:conv1_bits -s 1 -c 1 \
               -o gpurun_out/r1g_full_conv1 -f python tools/conv1_time.py 16384 > /dev/null 2>&1 ;;
    c3)    $B --config c3 > gpurun_out/plain_c3.log 2>&1 || exit 1
           ncu --set full --clock-control none --import-source on -k regex:env_solo_kernel_dungeon -s 3 -c 1 \
               -o gpurun_out/r1g_full_c3 -f $B --config c3 > /dev/null 2>&1 ;;
    *)     $B --config $what > gpurun_out/plain_$what.log 2>&1 || exit 1
           ncu --set full --clock-control none --import-source on -k regex:env_kernel -s 3 -c 1 \
               -o gpurun_out/r1g_full_$what -f $B --config $what > /dev/null 2>&1 ;;
  esac
done
echo done
