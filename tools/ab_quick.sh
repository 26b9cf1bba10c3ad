#!/bin/bash
# Quick A/B on one GPU box: build, the whole-solve GPU parity tests, bench lines without the CPU
# and e2e legs (per-kernel tables), written to gpurun_out/<tag>/.
tag=${1:-ab}; shift
cfgs=${@:-c4 c4j}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest exit $?"; tail -2 $out/pytest.log
for c in $cfgs; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
python tools/kernel_table.py $out/bench_*.json 2>/dev/null
