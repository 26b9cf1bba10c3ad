#!/bin/bash
# One gpurun call: GPU parity tests (fast subset unless FULL=1), then bench lines.
# usage: bash tools/gpu_quick.sh <tag> [configs...]
tag=$1; shift
mkdir -p gpurun_out
if [ -n "$FULL" ]; then sel="-m gpu"; else sel="-m gpu and not slow"; fi
timeout 900 python -m pytest tests -m "${sel#-m }" -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -3 gpurun_out/${tag}_pytest_gpu.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  python -c "import json,sys; d=json.load(open('gpurun_out/${tag}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', d['config']['rel_residual_dd']); [print('   %-22s %8.3f'%(k,v)) for k,v in d['roofline']['stage_ms_per_step'].items()]" || tail -5 gpurun_out/${tag}_bench_$c.err
done
if [ -x tools/microbench/fp64_mix ]; then tools/microbench/fp64_mix > gpurun_out/${tag}_fp64_mix.log 2>&1; cat gpurun_out/${tag}_fp64_mix.log; fi
