# round-2 final session E (final tree): C2 line, the other shapes, 2-rank ring, logical ring, K1 ncu at each point
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fe.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_c2_final4.json 2> gpurun_out/bench_c2_final4.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_final4.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['l'], d['config']['recall_at_10'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'], all(d['parity']['exact_visited_run']['counters_equal'].values()), 'cpu', d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])"
for c in c3s c4 c5s c2h c2g c2ivf; do
  timeout 1500 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_final4.json 2> gpurun_out/bench_${c}_final4.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_final4.json').read().strip().splitlines()[-1])
print('$c', d['value'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], d['config']['recall_at_10'], 'frac', d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['speedup_pathweaver_over_naive'], d['naive_sharded'].get('l'), d['naive_sharded'].get('recall_at_10'), 'ids', (d.get('parity') or {}).get('timed_lossy_run', {}).get('ids_equal_frac'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
PW_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2s --steps 5 --no-cpu > gpurun_out/bench_c2s_2ranks_final4.json 2> gpurun_out/bench_c2s_2ranks_final4.err; tail -c 400 gpurun_out/bench_c2s_2ranks_final4.json
for c in c3s c4 c5s; do
  read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_${c}_final4.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_${c}_final4 python tools/profile_run.py --config $c --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_${c}_final4.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_final4 python tools/profile_run.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_final4.log 2>&1
timeout 2400 python tools/logical_ring.py --config c2 --ns 2,4,8 --pw-grid 0.75:1,0.8:1 > gpurun_out/logical_c2_final4.jsonl 2> gpurun_out/logical_c2_final4.err; tail -3 gpurun_out/logical_c2_final4.jsonl | cut -c1-300
ls gpurun_out | grep final4 | wc -l
