#!/bin/bash
# round-2 evidence call: GPU suite, C4 bench line (per-kernel table), ncu launch list with DRAM bytes
tag=${1:-r2a}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -3 gpurun_out/${tag}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err
echo "bench exit $?"
python - <<PY
import json
d=json.load(open('gpurun_out/${tag}_bench_c4.json'))
r=d['roofline']
print('c4', round(d['ms_per_step'],3), 'ms', 'kernel', r['kernel'], round(r['frac'],3), r['bound'], 'fp64 in-run', r.get('fp64_peak_tflops_in_run'))
for k,v in sorted(r['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step']):
    print('   %-14s %7.3f ms  share %.3f  frac %s %s'%(k, v['ms_per_step'], v['share'], round(v.get('frac',0),3), v.get('bound')))
PY
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu exit $?"
