# Round session: tests, default bench (+ reference arm), launch list + ncu of K1,
# 2-rank dataflow ring on one GPU, the other configs.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/ref.json 2> gpurun_out/ref.err; cat gpurun_out/ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows" --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_${TAG:-x} python tools/profile_run.py --config c2 --l 256 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof.log 2>&1
PW_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2s --steps 5 --no-cpu > gpurun_out/bench_c2s_2ranks.json 2> gpurun_out/bench_c2s_2ranks.err; cat gpurun_out/bench_c2s_2ranks.json; tail -3 gpurun_out/bench_c2s_2ranks.err
for c in ${CONFIGS:-c5s}; do timeout 1500 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json; done
ls -la gpurun_out
