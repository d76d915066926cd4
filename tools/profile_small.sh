#!/bin/bash
# ncu captures of the c1 (64 envs, block mode) and c4 (64x64, lane team) step kernels
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-u8 --no-policy"
$B --config c1 > gpurun_out/plain_c1.log 2>&1 && $B --config c4 > gpurun_out/plain_c4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:env_solo_kernel_binary -s 3 -c 1 -o gpurun_out/r1d_full_c1 -f $B --config c1 > gpurun_out/ncu_c1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:env_kernel -s 3 -c 1 -o gpurun_out/r1d_full_c4 -f $B --config c4 > gpurun_out/ncu_c4.log 2>&1
echo done
