#!/bin/bash
# k_zs1 / k_zs2 occupancy A/B (LFDS_ZS_PAD1/2 force one CTA per SM): C4 per-kernel times and
# ncu DRAM bytes of the z-solvers
tag=${1:-zso}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
for pad in 0 120000; do
  LFDS_ZS_PAD1=$pad LFDS_ZS_PAD2=$pad timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${tag}_pad${pad}.json 2>&1
  python - <<PY
import json
d=json.load(open('gpurun_out/${tag}_pad${pad}.json'))
k=d['roofline']['kernels']
print('pad $pad', round(d['ms_per_step'],3), 'zs1', round(k['k_zs1']['ms_per_step'],3), 'zs2', round(k['k_zs2']['ms_per_step'],3))
PY
done
LFDS_ZS_PAD1=120000 LFDS_ZS_PAD2=120000 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_zs \
  --log-file gpurun_out/${tag}_ncu_pad.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_ncu.log 2>&1
python tools/launch_traffic.py c4 gpurun_out/${tag}_ncu_pad.csv
