timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
PW_LIB=tools/lib_prev.so timeout 900 python tools/ab.py --config c2 --l 256 2>>gpurun_out/ab.err >> gpurun_out/ab.log
timeout 900 python tools/ab.py --config c2 --l 256 2>>gpurun_out/ab.err >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
