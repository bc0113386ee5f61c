nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r02a.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02a.log
timeout 1500 python bench.py > gpurun_out/bench_c2_r02a.json 2> gpurun_out/bench_c2_r02a.err; tail -c 3000 gpurun_out/bench_c2_r02a.json
timeout 600 python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' > gpurun_out/ab_r02a.log 2>&1; cat gpurun_out/ab_r02a.log | tail -3
