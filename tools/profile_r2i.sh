tag=r2i
B="python bench.py --steps 2 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy"
$B > gpurun_out/plain_c5.log 2>&1 || { echo "plain c5 failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
bash tools/profile_r2.sh $tag c5 c3 c2 c5s
ls gpurun_out/ | grep $tag
