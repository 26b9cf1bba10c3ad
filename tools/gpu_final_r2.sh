#!/bin/bash
# Round-2 evidence in one gpurun call: GPU suite, smoke, bench lines of every workload, the
# reference arm, per-rank sharded compute, the C4 ncu launch list (time + DRAM bytes) and
# ncu --set full captures of the main kernels.  Everything lands in gpurun_out/<tag>/.
tag=${1:-final}
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
for c in c1 c2 c3 c4j c4q c5 c4h; do
  timeout 1200 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref exit $?"
SHARD_STAGES=1 timeout 900 python tools/shard_rank_time.py c4 2 4 8 > $out/shard_c4.log 2>&1
SHARD_STAGES=1 timeout 900 python tools/shard_rank_time.py c4q 8 > $out/shard_c4q.log 2>&1
cmd="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
$cmd > $out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches_c4.csv $cmd > $out/ncu_launches.log 2>&1
echo "ncu launches exit $?"
$cmd > $out/plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_xform3m|k_dstt|k_dstw|k_zs1|k_zs2|k_s5m|k_proj_rows" -c 12 \
  -o $out/prof_c4 $cmd > $out/ncu_full.log 2>&1
echo "ncu full exit $?"
