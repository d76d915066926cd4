#!/bin/bash
# r2 evidence for profiles/ (one B200, under gpurun):
#   1. ncu launch list of the c5 bench command (device time + DRAM bytes per launch)
#   2. --set full captures (digested on the box) of the c5/c3/c2/c4 step kernels,
#      the tcgen05 trunk kernel and the conv1 tile kernel
tag=${1:-r2}
B="python bench.py --steps 2 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy"
$B > gpurun_out/plain_c5.log 2>&1 || { echo "plain c5 failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
bash tools/profile_r2.sh $tag c5 c3 c2 c4
python tools/trunk_time.py 16384 > gpurun_out/plain_trunk.log 2>&1 || { echo "trunk failed"; exit 1; }
for k in trunk_kernel conv1_bits_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${tag}_full_$k -f python tools/trunk_time.py 65536 > gpurun_out/ncu_$k.log 2>&1
  python profiles/ncu_summary.py gpurun_out/${tag}_full_$k.ncu-rep 40 > gpurun_out/${tag}_ncu_$k.txt 2>&1
  ncu -i gpurun_out/${tag}_full_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src_$k.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/${tag}_src_$k.csv 50 > gpurun_out/${tag}_lines_$k.txt 2>&1
  rm -f gpurun_out/${tag}_src_$k.csv gpurun_out/${tag}_full_$k.ncu-rep
done
echo profile done
