#!/bin/bash
# warp-per-line step-2 solver (k_zsw) vs k_zs1: GPU parity subset, then C4 times and traffic
tag=${1:-zsw}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "shrunken or edge or uniform or modal or sine or graph or pass1" > gpurun_out/${tag}_pytest.log 2>&1
tail -3 gpurun_out/${tag}_pytest.log
for v in 0 1; do
  LFDS_ZSW=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${tag}_z$v.json 2>&1
  python - <<PY
import json
d=json.load(open('gpurun_out/${tag}_z$v.json'))
k=d['roofline']['kernels']
print('zsw $v', round(d['ms_per_step'],3), {n: (round(v['ms_per_step'],3), round(v.get('frac',0),3)) for n,v in k.items() if n in ('k_zs1','k_zsw','k_zs2')}, d['config']['rel_residual_dd'])
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_zs \
  --log-file gpurun_out/${tag}_ncu.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_ncu.log 2>&1
python tools/launch_traffic.py c4 gpurun_out/${tag}_ncu.csv
