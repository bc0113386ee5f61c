# final tree (round 2, session d): suite, smoke, C2 line, ncu at its point, launch list, e2e timeline
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fd.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final3.log 2>&1; tail -2 gpurun_out/pytest_gpu_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1; tail -1 gpurun_out/smoke_final3.log
timeout 1500 python bench.py > gpurun_out/bench_c2_final3.json 2> gpurun_out/bench_c2_final3.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_final3.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], d['config']['recall_at_10'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['roofline']['traffic'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'], d['parity']['exact_visited_run']['counters_equal'], 'cpu', d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_c2_final3.json 2> gpurun_out/ref_c2_final3.err; tail -c 400 gpurun_out/ref_c2_final3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows|init_run" --csv --log-file gpurun_out/launches_c2_final3.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu_final3.log 2>&1
ls gpurun_out | tail -3
