#!/bin/bash
tag=${1:-projb}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "shrunken or pass1 or edge or uniform" > gpurun_out/${tag}_pytest.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
for v in 0 1; do
  LFDS_PROJ_BULK=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${tag}_b$v.json 2>&1
  python - <<PY
import json
d=json.load(open('gpurun_out/${tag}_b$v.json'))
k=d['roofline']['kernels']
print('bulk $v', round(d['ms_per_step'],3), {n: (round(v['ms_per_step'],3), round(v.get('frac',0),3)) for n,v in k.items() if n.startswith('k_proj')}, d['config']['rel_residual_dd'])
PY
done
for c in c4j c4q c5; do
  for v in 0 1; do
  LFDS_PROJ_BULK=$v timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${tag}_${c}_b$v.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/${tag}_${c}_b$v.json')); k=d['roofline']['kernels']; print('$c bulk $v', round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if n.startswith('k_proj')})"
  done
done
