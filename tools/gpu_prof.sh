#!/bin/bash
# One gpurun call: ncu --set full captures (one launch each) of the named kernels, after a
# plain run of the same command.  Raw-metric and source CSVs are extracted on the box; a
# .ncu-rep is kept only if small (gpurun_out is capped at 64 MiB).
# usage: bash tools/gpu_prof.sh <tag> <config> <regex1> [<regex2> ...]
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
cmd="python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 300 $cmd > gpurun_out/${tag}_prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
i=0
for rx in "$@"; do
  i=$((i+1))
  out=/tmp/${tag}_k$i
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -c 1 -o $out $cmd \
     > gpurun_out/${tag}_prof_k${i}.log 2>&1
  ncu -i $out.ncu-rep --page raw --csv > gpurun_out/${tag}_prof_k${i}_raw.csv 2>/dev/null
  ncu -i $out.ncu-rep --page details --csv > gpurun_out/${tag}_prof_k${i}_details.csv 2>/dev/null
  ncu -i $out.ncu-rep --page source --csv > /tmp/src.csv 2>/dev/null && gzip -c /tmp/src.csv > gpurun_out/${tag}_prof_k${i}_source.csv.gz
  sz=$(stat -c %s $out.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -lt 8000000 ]; then cp $out.ncu-rep gpurun_out/; fi
done
du -sh gpurun_out
echo "exit 0"
