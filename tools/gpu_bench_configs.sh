# 1-GPU bench lines for the other BASELINE configs (C3 / C5 shard-sized, C4)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${CONFIGS:-c4 c3s c5s}; do
  timeout 1500 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "== $c"; cat gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err
done
