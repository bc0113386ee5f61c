# DGS query registers adopted: suite, smoke, C2 line
set -x
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_s18.log 2>&1; tail -3 gpurun_out/pytest_gpu_s18.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s18.log 2>&1; tail -1 gpurun_out/smoke_s18.log
timeout 1500 python bench.py > gpurun_out/bench_c2_s18.json 2> gpurun_out/bench_c2_s18.err; tail -c 300 gpurun_out/bench_c2_s18.json
