# K4 tensor-core kNN screen: first run (bounded), correctness + timing
timeout 420 python tools/knn_screen_probe.py --n 200000 --big 10000000 > gpurun_out/knn_probe_r02n.log 2>&1; tail -12 gpurun_out/knn_probe_r02n.log
