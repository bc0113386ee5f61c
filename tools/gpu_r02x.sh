# K4 with 8 epilogue warps: probe, exact tests, 10M build
timeout 420 python tools/knn_screen_probe.py --n 1000000 --big 10000000 --big-rows 37888 > gpurun_out/knn_probe_r02x.log 2>&1; tail -6 gpurun_out/knn_probe_r02x.log
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_cli.py -x -q -m gpu > gpurun_out/pytest_exact_r02x.log 2>&1; tail -3 gpurun_out/pytest_exact_r02x.log
timeout 1500 python tools/exact_build_probe.py --config c2 > gpurun_out/exact_build_c2_r02x.log 2>&1; tail -2 gpurun_out/exact_build_c2_r02x.log
