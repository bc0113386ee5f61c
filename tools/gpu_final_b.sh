# round-2 final session B: the other shapes, 2-rank ring, logical ring, K1 ncu at each point
set -x
for c in c3s c4 c5s c2h c2g c2ivf; do
  timeout 1500 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_final.json 2> gpurun_out/bench_${c}_final.err
  tail -c 300 gpurun_out/bench_${c}_final.json
done
PW_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2s --steps 5 --no-cpu > gpurun_out/bench_c2s_2ranks_final.json 2> gpurun_out/bench_c2s_2ranks_final.err; tail -c 300 gpurun_out/bench_c2s_2ranks_final.json
for c in c3s c4 c5s; do
  read L DR GI <<< $(python -c "import json;d=json.loads(open('gpurun_out/bench_${c}_final.json').read().strip().splitlines()[-1])['config'];print(d['l'],d['dgs_discard'],d['ghost_max_iter'])")
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_${c}_final python tools/profile_run.py --config $c --l $L --discard $DR --ghost-iter $GI --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_${c}_final.log 2>&1
done
timeout 2400 python tools/logical_ring.py --config c2 --ns 2,4,8 --pw-grid 0.75:1,0.8:1 > gpurun_out/logical_c2_final.jsonl 2> gpurun_out/logical_c2_final.err; cat gpurun_out/logical_c2_final.jsonl
