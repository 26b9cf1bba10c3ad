#!/bin/bash
# k_xplane variants (LFDS_XPLANE: 1 = CTA per plane at 2 CTAs per SM, 2 = warp per plane,
# 3 = CTA per plane at 3 CTAs per SM): parity tests per mode, then the C5 bench line per mode.
out=gpurun_out/xplane_modes
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
for x in 2 3 1; do
  LFDS_XPLANE=$x timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -s -k "plane_dense or shrunken_configs" > $out/pytest_x$x.log 2>&1
  echo "mode $x pytest exit $?"; grep -E "passed|failed" $out/pytest_x$x.log | tail -1
done
for x in 2 3 1 2 3 1; do
  LFDS_XPLANE=$x timeout 900 python bench.py --config c5 --no-cpu --no-e2e > $out/c5_x$x.json 2> $out/c5_x$x.err
  echo "bench c5 xplane=$x exit $?"
  python - <<PY
import json
d=json.load(open("$out/c5_x$x.json"))
k=d["roofline"]["kernels"]
print("c5 x=$x", round(d["ms_per_step"],3), {n:(round(v["ms_per_step"],3), round(v.get("frac",0),3)) for n,v in k.items() if n in ("k_xplane","k_xform")}, d["config"].get("rel_residual_dd"))
PY
done
