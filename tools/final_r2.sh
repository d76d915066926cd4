#!/bin/bash
# round-end evidence on one B200: GPU tests, smoke, every config's bench line,
# the reference arm, and the ncu launch list of the default bench command
tag=${1:-r2p}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${tag}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_ref_c5.json 2>&1; echo "ref c5 rc=$?"
for c in c1 c2 c3 c4; do
  timeout 400 python bench.py --config $c --no-policy > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err; echo "$c rc=$?"
done
B="python bench.py --steps 2 --warmup 3 --burn-in 0 --no-e2e --no-cpu-baseline --no-u8 --no-policy --no-proxy"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches_c5.csv $B > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launch list rc=$?"
