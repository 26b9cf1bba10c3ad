#!/bin/bash
# A/B of an environment knob on bench lines: tools/gpu_ab.sh <tag> "<VAR=a VAR=b ...>" <configs...>
# Builds, runs the fast GPU subset once (default env), then every config under every setting.
tag=$1; shift; settings=$1; shift
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest exit $?" >> $out/pytest.log; tail -2 $out/pytest.log
fi
for c in "$@"; do
  for s in $settings; do
    env $s timeout 600 python bench.py --config $c --no-cpu --no-e2e > $out/${c}_${s}.json 2> $out/${c}_${s}.err
    python - $out/${c}_${s}.json $c $s <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'FAILED', e); sys.exit()
ks=d['roofline'].get('kernels',{})
top=' '.join('%s=%.3f'%(k,v['ms_per_step']) for k,v in sorted(ks.items(), key=lambda kv:-kv[1]['ms_per_step'])[:6])
print(sys.argv[2], sys.argv[3], round(d['ms_per_step'],3), 'ms', d['config'].get('rel_residual_dd'), top)
PY
  done
done
