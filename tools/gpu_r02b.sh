# round 2: GPU tests on the new tree + ncu source capture of K1 at the C2 bench point
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r02b.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02b.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_r02b python tools/profile_run.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_r02b.log 2>&1
tail -2 gpurun_out/prof_c2_r02b.log; ls -la gpurun_out/*.ncu-rep
