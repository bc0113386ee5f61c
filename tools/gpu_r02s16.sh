# final tree: C3s line + K1 ncu at its point
set -x
timeout 1800 python bench.py --config c3s > gpurun_out/bench_c3s_s16.json 2> gpurun_out/bench_c3s_s16.err; tail -c 300 gpurun_out/bench_c3s_s16.json
read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_c3s_s16.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c3s_s16 python tools/profile_run.py --config c3s --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c3s_s16.log 2>&1
