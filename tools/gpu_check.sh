#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines, ncu launch list.
# usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${tag}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err
for c in c2 c3 c5; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 300 $cmd > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/${tag}_launches_c4.csv $cmd > gpurun_out/${tag}_ncu_launch.log 2>&1
echo done
