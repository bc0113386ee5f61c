timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
PW_LIB=tools/lib_prev.so timeout 900 python tools/ab.py --config c2 --l 256 --tuning '[{}, {"stage_rows":16,"visited_slots":2048}]' 2>>gpurun_out/ab.err >> gpurun_out/ab.log
timeout 900 python tools/ab.py --config c2 --l 256 --tuning '[{}, {"stage_rows":16,"visited_slots":64}, {"stage_rows":16,"visited_slots":256}, {"stage_rows":32,"visited_slots":64}, {"stage_rows":8,"visited_slots":64}]' 2>>gpurun_out/ab.err >> gpurun_out/ab.log
cat gpurun_out/ab.log
