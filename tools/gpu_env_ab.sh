#!/bin/bash
# A/B bench lines of one config under different environment settings / bench arguments (no tests).
# usage: bash tools/gpu_env_ab.sh <tag> <config> "VAR=a VAR2=b" "VAR=c|--plane-dst 0" ...
# (an item is "<env assignments>[|<extra bench.py arguments>]")
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
i=0
for item in "$@"; do
  i=$((i+1))
  envs=${item%%|*}; extra=""; [[ "$item" == *"|"* ]] && extra=${item#*|}
  env $envs timeout 600 python bench.py --config $cfg --no-cpu --no-e2e $extra > gpurun_out/${tag}_${cfg}_$i.json 2> gpurun_out/${tag}_${cfg}_$i.err
  python -c "import json; d=json.load(open('gpurun_out/${tag}_${cfg}_$i.json')); s=d['roofline']['stage_ms_per_step']; print('$cfg [$item]', round(d['ms_per_step'],3), 'ms', d['config']['rel_residual_dd'], ' '.join('%s=%.2f'%(k.replace('step',''),v) for k,v in s.items()))" || tail -3 gpurun_out/${tag}_${cfg}_$i.err
done
