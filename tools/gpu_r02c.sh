python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r02c.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02c.log
timeout 900 python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs tools/lib_r01.so,default --rounds 2 > gpurun_out/ab_r02c.log 2> gpurun_out/ab_r02c.err; cat gpurun_out/ab_r02c.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_r02c python tools/profile_run.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_r02c.log 2>&1
tail -1 gpurun_out/prof_c2_r02c.log
