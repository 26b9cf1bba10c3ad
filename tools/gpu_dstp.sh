#!/bin/bash
# persistent strided sine transform (k_dstp) vs k_dst: sine tests, then C4 per-kernel times
tag=${1:-dstp}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "sine or plane or uniform or edge or shrunken" > gpurun_out/${tag}_pytest.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
for v in 0 1; do
  LFDS_DST_PERSIST=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${tag}_p$v.json 2>&1
  python - <<PY
import json
d=json.load(open('gpurun_out/${tag}_p$v.json'))
k=d['roofline']['kernels']
print('persist $v', round(d['ms_per_step'],3), {n: round(k[n]['ms_per_step'],3) for n in ('k_dst','k_dstw')}, round(k['k_dst']['frac'],3))
PY
done
for c in c4j c4q; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${tag}_$c.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/${tag}_$c.json')); k=d['roofline']['kernels']; print('$c', round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.3})"
done
