# profile the current K1 at the C2 bench point: phase timers + ncu full capture
timeout 900 env PW_LIB=paper_2507_17094_b200/libpwb200_timers.so python tools/phase_timers.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' > gpurun_out/phase_c2_r02g.jsonl 2> gpurun_out/phase_c2_r02g.err; cat gpurun_out/phase_c2_r02g.jsonl; tail -2 gpurun_out/phase_c2_r02g.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_r02g python tools/profile_run.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_r02g.log 2>&1
tail -1 gpurun_out/prof_c2_r02g.log
