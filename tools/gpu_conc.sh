#!/bin/bash
# GPU tests, then bench lines with the two-stream block split off (LFDS_CONC=0) and on.
# usage: bash tools/gpu_conc.sh <tag> <configs...>
tag=$1; shift
mkdir -p gpurun_out
if [ -n "$FULL" ]; then sel="gpu"; else sel="gpu and not slow"; fi
timeout 900 python -m pytest tests -m "$sel" -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -2 gpurun_out/${tag}_pytest_gpu.log
for c in "$@"; do
  for cc in 0 1; do
    LFDS_CONC=$cc timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${tag}_${c}_conc$cc.json 2> gpurun_out/${tag}_${c}_conc$cc.err
    python -c "import json; d=json.load(open('gpurun_out/${tag}_${c}_conc$cc.json')); s=d['roofline']['stage_ms_per_step']; print('$c conc=$cc', round(d['ms_per_step'],3), 'ms', d['config']['rel_residual_dd'], ' '.join('%s=%.2f'%(k.replace('step',''),v) for k,v in s.items()))" || tail -3 gpurun_out/${tag}_${c}_conc$cc.err
  done
done
