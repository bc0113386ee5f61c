# full GPU suite + smoke on the current tree
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02y.log 2>&1 || { tail -20 gpurun_out/build_r02y.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_r02y.log 2>&1; tail -15 gpurun_out/pytest_gpu_r02y.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02y.log 2>&1; tail -2 gpurun_out/smoke_r02y.log
