#!/bin/bash
# every BASELINE config through bench.py (builder lines for profiles/) + the reference arm
tag=${1:-r2}
for c in c1 c2 c3 c4; do
  python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err; echo "$c rc=$?"
  python bench.py --config $c --impl reference > gpurun_out/${tag}_bench_ref_$c.json 2>&1; echo "ref $c rc=$?"
done
python bench.py --impl reference > gpurun_out/${tag}_bench_ref_c5.json 2>&1; echo "ref c5 rc=$?"
