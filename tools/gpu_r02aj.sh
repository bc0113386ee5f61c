PW_UPLOAD_DEBUG=1 timeout 1500 python bench.py > gpurun_out/bench_c2_r02aj.json 2> gpurun_out/bench_c2_r02aj.err; grep -E "pw_run upload|Error" gpurun_out/bench_c2_r02aj.err | head -5; python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_r02aj.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config']['l'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'], 'cpu', d['cpu_baseline']['value'], d['clocks'])"
