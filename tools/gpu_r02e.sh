# round 2 re-entry: GPU suite + default bench on the restored tree
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r02e.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02e.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02e.log 2>&1; tail -2 gpurun_out/smoke_r02e.log
timeout 1500 python bench.py > gpurun_out/bench_c2_r02e.json 2> gpurun_out/bench_c2_r02e.err; tail -c 4000 gpurun_out/bench_c2_r02e.json; tail -5 gpurun_out/bench_c2_r02e.err
