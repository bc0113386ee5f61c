# Round-end measurement session: bench lines for every config, the reference
# arm, and ncu captures of K1 at each config's chosen operating point.
set -x
for c in c2 c4 c3s c5s; do
  if [ $c = c2 ]; then timeout 1200 python bench.py > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  else timeout 1200 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; fi
  read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_final_$c python tools/profile_run.py --config $c --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_final_$c.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill_kernel|gather_rows" --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
ls -la gpurun_out
