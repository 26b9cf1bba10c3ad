#!/bin/bash
# Round-end evidence: bench lines (all configs), ncu launch list of the default bench, and
# ncu --set full captures of the main kernels (raw CSV + source CSV kept under gpurun_out).
tag=${1:-r01final}
mkdir -p gpurun_out
for c in c4 c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 300 $cmd > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/${tag}_launches_c4.csv $cmd > gpurun_out/${tag}_ncu_launch.log 2>&1
echo done
