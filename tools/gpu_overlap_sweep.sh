#!/bin/bash
# Sweep of the concurrent-transform knobs on one config: LFDS_OVERLAP, LFDS_SINE_CTAS, LFDS_DENSE_CTAS.
# usage: bash tools/gpu_overlap_sweep.sh <tag> <config> "<ov> <sine> <dense>" ...
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -2 gpurun_out/${tag}_pytest_gpu.log
for combo in "$@"; do
  set -- $combo
  LFDS_OVERLAP=$1 LFDS_SINE_CTAS=$2 LFDS_DENSE_CTAS=$3 timeout 600 python bench.py --config $cfg --no-cpu --no-e2e \
     > gpurun_out/${tag}_${cfg}_$1_$2_$3.json 2> gpurun_out/${tag}_${cfg}_$1_$2_$3.err
  python -c "import json,sys; d=json.load(open('gpurun_out/${tag}_${cfg}_$1_$2_$3.json')); s=d['roofline']['stage_ms_per_step']; print('ov=$1 sine=$2 dense=$3', round(d['ms_per_step'],3), 'ms', d['config']['rel_residual_dd'], ' '.join('%s=%.2f'%(k.replace('step',''),v) for k,v in s.items() if 'sine' in k or 'dense' in k))" || tail -3 gpurun_out/${tag}_${cfg}_$1_$2_$3.err
done
