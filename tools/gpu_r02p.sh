timeout 420 python tools/knn_screen_probe.py --n 1000000 --big 10000000 --big-rows 37888 > gpurun_out/knn_probe_r02p.log 2>&1; tail -8 gpurun_out/knn_probe_r02p.log
