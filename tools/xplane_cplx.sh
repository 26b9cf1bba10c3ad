#!/bin/bash
# k_xplane with complex-basis axes (C x R, R x C, C x C blocks of at most 32 nodes): the whole GPU
# parity file, then bench lines of the configs whose block routing changed, against LFDS_XPLANE=0.
out=gpurun_out/xplane_cplx
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py tests/test_gpu_hetero.py -m gpu -q -p no:cacheprovider -s > $out/pytest.log 2>&1
echo "pytest exit $?" >> $out/pytest.log
grep -E "passed|failed" $out/pytest.log | tail -2
for c in c5 c3 c2 c4q c4j; do
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
