# HEAD at the end of round 2: build, suite, smoke, C2 line, reference arm
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s26.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_s26.log 2>&1; tail -3 gpurun_out/pytest_gpu_s26.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s26.log 2>&1; tail -1 gpurun_out/smoke_s26.log
timeout 1500 python bench.py > gpurun_out/bench_c2_s26.json 2> gpurun_out/bench_c2_s26.err; tail -c 300 gpurun_out/bench_c2_s26.json
timeout 1500 python bench.py --impl reference --steps 2 > gpurun_out/ref_c2_s26.json 2> gpurun_out/ref_c2_s26.err; tail -c 300 gpurun_out/ref_c2_s26.json
