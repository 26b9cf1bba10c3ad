#!/bin/bash
# ncu --set full of one kernel kind in the C4 bench: tools/gpu_prof_k.sh <tag> <regex> [count] [config]
tag=$1; rx=$2; cnt=${3:-2}; cfg=${4:-c4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
cmd="python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu --no-e2e"
$cmd > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$rx -c $cnt -o gpurun_out/${tag} $cmd > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu exit $?"
