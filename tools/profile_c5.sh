#!/bin/bash
# c5 launch list (device time + DRAM bytes per launch) and one --set full capture of the step kernel
tag=${1:-r1e}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-graph"
$B > gpurun_out/plain_c5.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:env_solo_kernel_binary -s 3 -c 1 \
    -o gpurun_out/${tag}_full_c5 -f $B > gpurun_out/ncu_c5.log 2>&1
echo done
