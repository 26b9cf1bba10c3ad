#!/bin/bash
# Maxwell z-solve A/B: parity tests, then the mw1 bench at 4 and 3 CTAs per SM (LFDS_MW_MINB).
out=gpurun_out/${1:-mw_ab}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_maxwell.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest exit $?"; tail -2 $out/pytest.log
for mb in 4 3; do
  LFDS_MW_MINB=$mb timeout 600 python tools/mw_bench.py --two-level 2 4 > $out/mw1_minb$mb.json 2> $out/mw1_minb$mb.err
  echo "minb $mb exit $?"
  python - $out/mw1_minb$mb.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d["kernels"]["k_mw_zsolve"]
print(sys.argv[1], "solve", round(d["ms_per_step"], 3), "ms; k_mw_zsolve", round(k["ms"], 3), "ms frac", round(k["frac"], 3),
      "two-level", {b: round(v["ms"], 2) for b, v in d.get("two_level", {}).items()})
PY
done
