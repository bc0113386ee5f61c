# K4 streamed query block (d > 128): exact-build tests, throughput at d = 200 / 96
set -x
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q > gpurun_out/pytest_exact_s5.log 2>&1; tail -3 gpurun_out/pytest_exact_s5.log
timeout 600 python tools/knn_screen_probe.py --n 200000 --d 200 --big 2000000 > gpurun_out/knn_probe_d200_s5.log 2>&1; tail -8 gpurun_out/knn_probe_d200_s5.log
timeout 600 python tools/knn_screen_probe.py --n 200000 --d 96 --big 2000000 --only-throughput > gpurun_out/knn_probe_d96_s5.log 2>&1; tail -4 gpurun_out/knn_probe_d96_s5.log
