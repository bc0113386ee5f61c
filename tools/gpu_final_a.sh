# round-2 final session A: suite, smoke, C2 line + reference arm, ncu + launch list at the C2 point
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fa.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -1 gpurun_out/smoke_final.log
timeout 1500 python bench.py > gpurun_out/bench_c2_final.json 2> gpurun_out/bench_c2_final.err; tail -c 400 gpurun_out/bench_c2_final.json
timeout 1500 python bench.py --impl reference --steps 2 > gpurun_out/ref_c2_final.json 2> gpurun_out/ref_c2_final.err; tail -c 300 gpurun_out/ref_c2_final.json
read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_c2_final.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_final python tools/profile_run.py --config c2 --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows" --csv --log-file gpurun_out/launches_c2_final.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu_final.log 2>&1
ls -la gpurun_out | tail -5
