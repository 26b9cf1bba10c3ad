#!/bin/bash
# Evidence of the k_xplane code in one gpurun call: GPU suite, smoke, bench lines (default C4 and the
# configs with plane-dense blocks), C5 launch list (time + DRAM bytes), ncu --set full of k_xplane.
tag=${1:-final4}
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
for c in c5 c3 c2 c1; do
  timeout 1200 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
cmd="python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-e2e"
$cmd > $out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -c 3000 \
  --log-file $out/launches_c5.csv $cmd > $out/ncu_launches.log 2>&1
echo "ncu launches exit $?"
$cmd > $out/plain2_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_xplane" -c 2 \
  -o $out/prof_xplane $cmd > $out/ncu_full.log 2>&1
echo "ncu full exit $?"
ncu -i $out/prof_xplane.ncu-rep --page raw --csv > $out/ncu_k_xplane_raw.csv 2>/dev/null
