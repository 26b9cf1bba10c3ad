out=gpurun_out/xsmall2; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
for x in 1 0; do
  LFDS_XSMALL=$x timeout 600 python bench.py --config c5 --no-cpu --no-e2e > $out/c5_x$x.json 2> $out/c5_x$x.err; echo "c5 x$x exit $?"
  python tools/kernel_table.py $out/c5_x$x.json 2>/dev/null | head -3
done
