timeout 1500 python tools/exact_build_probe.py --config c2 --compare-ivf > gpurun_out/exact_build_c2_r02q.log 2>&1; tail -5 gpurun_out/exact_build_c2_r02q.log
