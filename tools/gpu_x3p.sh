#!/bin/bash
tag=${1:-x3p}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "shrunken or uniform or modal or graph or pass1 or tma" > gpurun_out/${tag}_pytest.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
for v in 0 1; do
  LFDS_X3P=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${tag}_x$v.json 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/${tag}_x$v.json').read().strip().splitlines()[-1])
k=d['roofline']['kernels']
print('x3p $v', round(d['ms_per_step'],3), {n: (round(v['ms_per_step'],3), round(v.get('frac',0),3)) for n,v in k.items() if n.startswith('k_xform')}, d['config']['rel_residual_dd'])
PY
done
for c in c4q c3 c5; do
  for v in 0 1; do
  LFDS_X3P=$v timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${tag}_${c}_x$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/${tag}_${c}_x$v.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$c x3p $v', round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if n.startswith('k_xform')})"
  done
done
