timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r02af.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02af.log
timeout 1500 python bench.py > gpurun_out/bench_c2_r02af.json 2> gpurun_out/bench_c2_r02af.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_r02af.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'], 'cpu', d['cpu_baseline']['value'], d['clocks'])"; tail -2 gpurun_out/bench_c2_r02af.err
