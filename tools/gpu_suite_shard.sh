#!/bin/bash
tag=${1:-ss}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
grep -E "passed|failed|FAILED|rel residual" gpurun_out/${tag}_pytest_gpu.log | tail -8
SHARD_STAGES=1 timeout 900 python tools/shard_rank_time.py c4 2 4 8 > gpurun_out/${tag}_shard_c4.log 2>&1
grep -v "^{" gpurun_out/${tag}_shard_c4.log
