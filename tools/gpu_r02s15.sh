# final tree: suite, smoke, C2 line, reference arm, launch list, 2 ranks on one GPU
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s15.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_s15.log 2>&1; tail -3 gpurun_out/pytest_gpu_s15.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s15.log 2>&1; tail -1 gpurun_out/smoke_s15.log
timeout 1500 python bench.py > gpurun_out/bench_c2_s15.json 2> gpurun_out/bench_c2_s15.err; tail -c 300 gpurun_out/bench_c2_s15.json
timeout 1500 python bench.py --impl reference --steps 2 > gpurun_out/ref_c2_s15.json 2> gpurun_out/ref_c2_s15.err; tail -c 300 gpurun_out/ref_c2_s15.json
env | grep -c CUDA_INJECTION64_PATH; ncu --print-summary none bash -c 'env | grep -c CUDA_INJECTION64_PATH' 2>/dev/null | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows|init_run" --csv --log-file gpurun_out/launches_c2_s15.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu_s15.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --config c2s --no-cpu > gpurun_out/bench_c2s_2ranks_s15.json 2> gpurun_out/bench_c2s_2ranks_s15.err; tail -c 300 gpurun_out/bench_c2s_2ranks_s15.json
