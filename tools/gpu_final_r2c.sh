#!/bin/bash
# Evidence of the final k_xplane code (real and complex bases) in one gpurun call: GPU suite, smoke,
# bench lines of every BJ config and partition variant, the C5 A/B against LFDS_XPLANE=0, and an
# ncu --set full capture of k_xplane.
tag=${1:-final5}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
nvidia-smi > $out/nvidia_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $out/pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> $out/pytest_gpu.log
grep -E "passed|failed" $out/pytest_gpu.log | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
for c in c5 c3 c2 c1 c4q c4j; do
  timeout 1200 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
for c in c5 c3 c4q; do
  LFDS_XPLANE=0 timeout 900 python bench.py --config $c --no-cpu --no-e2e > $out/bench_${c}_x0.json 2> $out/bench_${c}_x0.err; echo "bench $c x0 exit $?"
done
python - <<PY
import json
for c in ("c4","c5","c5_x0","c3","c3_x0","c2","c1","c4q","c4q_x0","c4j"):
    try:
        d=json.load(open("$out/bench_%s.json" % c))
        k=d["roofline"]["kernels"]
        print(c, round(d["ms_per_step"],3), {n:(round(v["ms_per_step"],3), round(v.get("frac",0),3)) for n,v in k.items() if n in ("k_xplane","k_xform","k_xform3m")}, d["config"].get("rel_residual_dd"))
    except Exception as e:
        print(c, "ERR", e)
PY
cmd="python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-e2e"
$cmd > $out/plain2_c5.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_xplane" -c 4 \
  -o $out/prof_xplane $cmd > $out/ncu_full.log 2>&1
echo "ncu full exit $?"
ncu -i $out/prof_xplane.ncu-rep --page raw --csv > $out/ncu_k_xplane_raw.csv 2>/dev/null
