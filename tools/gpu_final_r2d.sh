#!/bin/bash
# Final check of the plan-level k_xplane gate: GPU suite, smoke, bench lines of every config.
tag=${1:-final6}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $out/pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> $out/pytest_gpu.log
grep -E "passed|failed" $out/pytest_gpu.log | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
for c in c5 c3 c2 c1 c4q c4j; do
  timeout 1200 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
python - <<PY
import json
for c in ("c4","c5","c3","c2","c1","c4q","c4j"):
    try:
        d=json.load(open("$out/bench_%s.json" % c))
        k=d["roofline"]["kernels"]
        print(c, round(d["ms_per_step"],3), {n:(round(v["ms_per_step"],3), round(v.get("frac",0),3)) for n,v in k.items() if n in ("k_xplane","k_xform","k_xform3m")}, d["config"].get("rel_residual_dd"))
    except Exception as e:
        print(c, "ERR", e)
PY
