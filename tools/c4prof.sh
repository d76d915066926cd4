B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-u8 --config c4"
for t in 64 32; do LG_TEAM_THREADS=$t python bench.py --config c4 --no-e2e --no-cpu-baseline --no-u8 | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('threads $t', d['value']/1e6, d['roofline']['step_kernel_ms'])"; done
$B > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:env_kernel -s 3 -c 1 -o gpurun_out/r1c_full_c4 -f $B > gpurun_out/ncu_c4.log 2>&1; tail -2 gpurun_out/ncu_c4.log
