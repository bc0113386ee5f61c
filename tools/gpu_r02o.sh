# K4 screen: where does the time go (debug probes) + ncu of one launch
for dbg in 0 1 2 3; do PW_KNN_DEBUG=$dbg timeout 300 python tools/knn_screen_probe.py --n 1000000 --big-rows 37888 2>&1 | grep throughput | sed "s/^/dbg=$dbg /"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_screen -c 1 -o gpurun_out/prof_knn_r02o python tools/knn_screen_probe.py --n 200000 --big-rows 18944 > gpurun_out/prof_knn_r02o.log 2>&1; tail -2 gpurun_out/prof_knn_r02o.log
