# runtime-knob A/B at the C2 (exact graph) bench point
timeout 1500 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '[{"flags": 2}, {"flags": 3}, {"flags": 6}, {"flags": 2, "visited_slots": 2048}, {"flags": 2, "visited_slots": 8192}, {"flags": 2, "stage_rows": 20}, {"flags": 2, "stage_rows": 12}]' --rounds 2 > gpurun_out/ab_knobs_r02v.log 2> gpurun_out/ab_knobs_r02v.err; python -c "
import json
for l in open('gpurun_out/ab_knobs_r02v.log'):
    d=json.loads(l); print(d['round'], d['tuning'], 'naive', d['naive']['kernel_ms'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['warps'])"; tail -2 gpurun_out/ab_knobs_r02v.err
timeout 2400 python tools/logical_ring.py --config c2 --ns 8 --pw-grid 0.8:1 > gpurun_out/logical_c2x_dc_r02v.jsonl 2> gpurun_out/logical_c2x_dc_r02v.err; cat gpurun_out/logical_c2x_dc_r02v.jsonl
for c in c2h c2g; do
  timeout 1500 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_r02v.json 2> gpurun_out/bench_${c}_r02v.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_r02v.json').read().strip().splitlines()[-1])
print('$c', d['value'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], d['config']['recall_at_10'], 'frac', d['roofline']['frac'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['l'], d['naive_sharded']['recall_at_10'])
"; tail -2 gpurun_out/bench_${c}_r02v.err | cut -c1-400
done
