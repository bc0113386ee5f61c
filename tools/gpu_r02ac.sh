# C2 line with the FAST K1 + ncu capture of it
timeout 1500 python bench.py > gpurun_out/bench_c2_r02ac.json 2> gpurun_out/bench_c2_r02ac.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_r02ac.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'], d['parity']['exact_visited_run']['counters_equal'], 'cpu', d['cpu_baseline']['value'], d['clocks'])"
read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_c2_r02ac.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_r02ac python tools/profile_run.py --config c2 --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_r02ac.log 2>&1; tail -1 gpurun_out/prof_c2_r02ac.log
