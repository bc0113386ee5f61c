# C5s on the exact graph (K4 streamed query block) + K1 ncu at its point; C4 with the K4-built graph
set -x
timeout 1800 python bench.py --config c5s > gpurun_out/bench_c5s_s6.json 2> gpurun_out/bench_c5s_s6.err; tail -c 600 gpurun_out/bench_c5s_s6.json
read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_c5s_s6.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c5s_s6 python tools/profile_run.py --config c5s --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c5s_s6.log 2>&1
timeout 1200 python bench.py --config c4 > gpurun_out/bench_c4_s6.json 2> gpurun_out/bench_c4_s6.err; tail -c 400 gpurun_out/bench_c4_s6.json
