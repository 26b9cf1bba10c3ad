#!/bin/bash
# Round evidence on one GPU: bench lines of every config (with e2e and the CPU oracle
# baseline), the --impl reference line, the ncu launch list of the default bench command, and
# ncu --set full captures (one launch each) of the main kernels of the default config (the
# residual kernel on C2, the plane sine transform on C4q).
tag=${1:-r01ev}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log; tail -2 gpurun_out/${tag}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/${tag}_smoke.log
for c in c4 c1 c2 c3 c5 c4j c4q c4h; do
  timeout 1200 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/${tag}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', '%.3e'%d['value'], 'e2e', d['e2e'] and '%.3e'%d['e2e']['value'], 'cpu', d['cpu_baseline'] and '%.3e'%d['cpu_baseline']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), 'solve', round(d['roofline']['solve']['frac'],3))" || tail -3 gpurun_out/${tag}_bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; tail -c 400 gpurun_out/${tag}_bench_ref.json
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 300 $cmd > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/${tag}_launches_c4.csv $cmd > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launch list exit $?"
cmd1="python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu"
i=0
for rx in "k_zs2" "k_s5m" "k_zs1" "k_dstw" "k_dst<" "k_xform3m" "k_proj_rows" "k_residual" "k_dst2"; do
  i=$((i+1))
  c=$cmd1; [ "$rx" = "k_residual" ] && c="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu"
  [ "$rx" = "k_dst2" ] && c="python bench.py --config c4q --steps 1 --warmup 0 --no-e2e --no-cpu"
  out=/tmp/${tag}_k$i
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -c 1 -o $out $c > gpurun_out/${tag}_prof_k${i}.log 2>&1
  ncu -i $out.ncu-rep --page raw --csv > gpurun_out/${tag}_prof_k${i}_raw.csv 2>/dev/null
  ncu -i $out.ncu-rep --page source --csv > /tmp/src.csv 2>/dev/null && gzip -c /tmp/src.csv > gpurun_out/${tag}_prof_k${i}_source.csv.gz
done
du -sh gpurun_out
