#!/bin/bash
# GPU tests (fast subset) + bench lines incl. the phased (block-sharded) path at N=1.
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -3 gpurun_out/${tag}_pytest_gpu.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  python -c "import json,sys; d=json.load(open('gpurun_out/${tag}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', d['config']['rel_residual_dd'], 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'solve-roof', round(d['roofline']['solve']['frac'],3)); [print('   %-22s %8.3f'%(k,v)) for k,v in d['roofline']['stage_ms_per_step'].items()]" || tail -5 gpurun_out/${tag}_bench_$c.err
done
timeout 600 python bench.py --config c4 --no-cpu --shard blocks > gpurun_out/${tag}_bench_c4_phased.json 2> gpurun_out/${tag}_bench_c4_phased.err
python -c "import json; d=json.load(open('gpurun_out/${tag}_bench_c4_phased.json')); print('c4 phased', round(d['ms_per_step'],3), d['config']['rel_residual_dd'], d['e2e'])" || tail -5 gpurun_out/${tag}_bench_c4_phased.err
