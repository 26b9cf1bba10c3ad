#!/bin/bash
# GPU suite only: tools/gpu_tests.sh <tag> [pytest -k expr]
tag=${1:-t}; k=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail gpurun_out/${tag}_build.log; exit 1; }
if [ -n "$k" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "$k" > gpurun_out/${tag}_pytest_gpu.log 2>&1
else
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/${tag}_pytest_gpu.log 2>&1
fi
echo "pytest gpu exit $?" >> gpurun_out/${tag}_pytest_gpu.log
grep -E "passed|failed|error|FAILED|rel2" gpurun_out/${tag}_pytest_gpu.log | tail -60
