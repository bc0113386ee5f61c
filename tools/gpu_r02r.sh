timeout 420 python tools/knn_screen_probe.py --n 1000000 --big 10000000 --big-rows 37888 > gpurun_out/knn_probe_r02r.log 2>&1; tail -8 gpurun_out/knn_probe_r02r.log
timeout 1500 python tools/exact_build_probe.py --config c2 > gpurun_out/exact_build_c2_r02r.log 2>&1; tail -3 gpurun_out/exact_build_c2_r02r.log
