#!/bin/bash
tag=${1:-dstt}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "sine or plane or uniform or shrunken or graph" > gpurun_out/${tag}_pytest.log 2>&1
tail -3 gpurun_out/${tag}_pytest.log
for v in 0 1; do
  timeout 600 python bench.py --no-cpu --no-e2e --dst-tma $v > gpurun_out/${tag}_t$v.json 2>&1
  python - <<PY
import json
d=json.load(open('gpurun_out/${tag}_t$v.json'))
k=d['roofline']['kernels']
print('tma $v', round(d['ms_per_step'],3), {n: (round(v['ms_per_step'],3), round(v.get('frac',0),3)) for n,v in k.items() if n.startswith('k_dst')}, d['config']['rel_residual_dd'])
PY
done
for c in c4j c3; do
  for v in 0 1; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --dst-tma $v > gpurun_out/${tag}_${c}_t$v.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/${tag}_${c}_t$v.json')); k=d['roofline']['kernels']; print('$c tma $v', round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if n.startswith('k_dst')})"
  done
done
