# round-2 session 4: ncu --set full of K1 at the C2 point on HEAD + phase timers
set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_c2_s4 python tools/profile_run.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --reps 3 --tuning '{"flags": 2}' > gpurun_out/prof_c2_s4.log 2>&1
PW_LIB=paper_2507_17094_b200/libpwb200_timers.so timeout 900 python tools/phase_timers.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' > gpurun_out/phase_c2_s4.jsonl 2> gpurun_out/phase_c2_s4.err
tail -3 gpurun_out/phase_c2_s4.jsonl
ls -la gpurun_out | tail -5
