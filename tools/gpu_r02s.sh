# C2 on the exact graph (K4-built): bench line, K1 ncu capture at its point, logical ring 2/4/8
timeout 1500 python bench.py > gpurun_out/bench_c2_r02s.json 2> gpurun_out/bench_c2_r02s.err; tail -c 600 gpurun_out/bench_c2_r02s.json; grep -E "index built|pathweaver discard|naive" gpurun_out/bench_c2_r02s.err | tail -20
read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_c2_r02s.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_r02s python tools/profile_run.py --config c2 --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_r02s.log 2>&1; tail -1 gpurun_out/prof_c2_r02s.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows" --csv --log-file gpurun_out/launches_c2_r02s.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu_r02s.log 2>&1
timeout 2400 python tools/logical_ring.py --config c2 --ns 2,4,8 --ext --pw-grid 0.75:1,0.8:1,0.7:1 > gpurun_out/logical_c2x_r02s.jsonl 2> gpurun_out/logical_c2x_r02s.err; python -c "
import json
for l in open('gpurun_out/logical_c2x_r02s.jsonl'):
    d=json.loads(l); print(d['n_shards'], d['naive'], d['pathweaver'], d.get('pw_over_naive'), d.get('extension_best'), d.get('ext_over_naive'))"
