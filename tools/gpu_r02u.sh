# round-2 bench lines: C3s (exact graph, u8), C4, C5s, c2h, c2g, 2-rank dataflow ring (NVLink fields), reference arm
for c in c3s c4 c5s c2h c2g; do
  timeout 1500 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_r02u.json 2> gpurun_out/bench_${c}_r02u.err
  python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/bench_${c}_r02u.json').read().strip().splitlines()[-1])
    print('$c', d['value'], d['e2e']['value'], d['config']['l'], d['config']['dgs_discard'], d['config']['ghost_max_iter'], d['config']['recall_at_10'], 'frac', d['roofline']['frac'], 'naive', d['naive_sharded']['value'], d['naive_sharded']['l'], d['naive_sharded']['recall_at_10'], 'ids', d['parity']['timed_lossy_run']['ids_equal_frac'] if d.get('parity') else None, 'build', d['config']['index_build_s'])
except Exception as e: print('$c failed', e)
"; tail -2 gpurun_out/bench_${c}_r02u.err
done
PW_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2s --steps 5 --no-cpu > gpurun_out/bench_c2s_2ranks_r02u.json 2> gpurun_out/bench_c2s_2ranks_r02u.err; tail -c 800 gpurun_out/bench_c2s_2ranks_r02u.json; tail -3 gpurun_out/bench_c2s_2ranks_r02u.err
timeout 1500 python bench.py --impl reference --steps 2 > gpurun_out/ref_c2_r02u.json 2> gpurun_out/ref_c2_r02u.err; tail -c 1500 gpurun_out/ref_c2_r02u.json
