#!/bin/bash
tag=${1:-shard}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "sharded or nccl or pass1" > gpurun_out/${tag}_pytest.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
SHARD_STAGES=1 timeout 900 python tools/shard_rank_time.py c4 2 4 8 > gpurun_out/${tag}_c4.log 2>&1
grep -v "^{" gpurun_out/${tag}_c4.log
