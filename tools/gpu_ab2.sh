#!/bin/bash
# Build, fast GPU parity subset (defaults), then kernel tables of configs under env settings.
# usage: tools/gpu_ab2.sh <tag> "<cfgs>" "<setting1>" "<setting2>" ...   (setting: "VAR=a VAR2=b" or "-")
tag=$1; cfgs=$2; shift 2
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest exit $?"; tail -2 $out/pytest.log
fi
for c in $cfgs; do
  for s in "$@"; do
    n=$(echo "$s" | tr ' =' '__')
    [ "$s" = "-" ] && s=""
    env $s timeout 600 python bench.py --config $c --no-cpu --no-e2e > $out/${c}_$n.json 2> $out/${c}_$n.err
    python - $out/${c}_$n.json "$c [$s]" <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print(sys.argv[2], 'FAILED', e); sys.exit()
ks=d['roofline'].get('kernels',{})
top=' '.join('%s=%.3f'%(k,v['ms_per_step']) for k,v in sorted(ks.items(), key=lambda kv:-kv[1]['ms_per_step'])[:8])
print(sys.argv[2], round(d['ms_per_step'],3), 'ms', '%.2e'%d['config'].get('rel_residual_dd'), top)
PY
  done
done
