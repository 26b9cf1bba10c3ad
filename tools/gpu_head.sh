#!/bin/bash
# Verify HEAD on a B200: build, full GPU suite, smoke, C4 bench line.  usage: tools/gpu_head.sh <tag>
tag=${1:-head}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
python tools/results_table.py $out 2>/dev/null | tail -3
