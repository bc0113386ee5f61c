# final tree: suite, smoke, C2 line, ncu at its point, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final2.log 2>&1; tail -2 gpurun_out/pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; tail -1 gpurun_out/smoke_final2.log
timeout 1500 python bench.py > gpurun_out/bench_c2_final2.json 2> gpurun_out/bench_c2_final2.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_final2.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], d['config']['recall_at_10'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['roofline']['traffic'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'], d['parity']['exact_visited_run']['counters_equal'], 'cpu', d['cpu_baseline']['value'], d['clocks'])"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_final2 python tools/profile_run.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_final2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows" --csv --log-file gpurun_out/launches_c2_final2.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu_final2.log 2>&1
ls gpurun_out | tail -3
