# round-1 evidence: tests, bench (C2), reference arm, ncu launch list + full capture
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; cat gpurun_out/ref_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --config c2 --l 256 --reps 3 > gpurun_out/launches_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_r01 python tools/profile_run.py --config c2 --l 256 > gpurun_out/prof_r01.log 2>&1; tail -1 gpurun_out/prof_r01.log
