#!/bin/bash
# A/B of the plane dense transform k_xplane (LFDS_XPLANE=0: x pass + y pass through k_xsmall):
# the new parity test, the shrunken-config parity tests, then C5 / C3 / C2 bench lines both ways.
out=gpurun_out/xplane
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -s -k "plane_dense or shrunken or graph_replay or sharded_solve" > $out/pytest.log 2>&1
echo "pytest exit $?" >> $out/pytest.log
grep -E "passed|failed|rel2" $out/pytest.log | tail -12
for c in c5 c3 c2; do
  for x in 1 0; do
    LFDS_XPLANE=$x timeout 900 python bench.py --config $c --no-cpu --no-e2e > $out/${c}_x$x.json 2> $out/${c}_x$x.err
    echo "bench $c xplane=$x exit $?"
    python - <<PY
import json
d=json.load(open("$out/${c}_x$x.json"))
k=d["roofline"]["kernels"]
print("$c x=$x", round(d["ms_per_step"],3), {n:(round(v["ms_per_step"],3), round(v.get("frac",0),3)) for n,v in k.items() if n in ("k_xplane","k_xform","k_xform3m")}, d["config"].get("rel_residual_dd"))
PY
  done
done
