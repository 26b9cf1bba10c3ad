#!/bin/bash
# Extra evidence: ncu launch lists (time + DRAM bytes) of the C4j / C4q steps and a full capture of
# the Maxwell z-solve.  Everything lands in gpurun_out/<tag>/.
tag=${1:-extra}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || exit 1
for c in c4j c4q; do
  cmd="python bench.py --config $c --steps 1 --warmup 1 --no-cpu --no-e2e"
  $cmd > $out/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches_$c.csv $cmd > $out/ncu_launches_$c.log 2>&1
  echo "launches $c exit $?"
done
cmd="python tools/mw_bench.py --steps 1 --warmup 1"
$cmd > $out/mw_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mw_zsolve" -c 1 -o $out/prof_mw $cmd > $out/ncu_mw.log 2>&1
echo "mw ncu exit $?"
