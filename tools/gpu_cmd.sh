timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for L in tools/libpwb200_v1.so paper_2507_17094_b200/libpwb200.so; do
  PW_LIB=$L timeout 300 python tools/ab.py --config c2s 2>>gpurun_out/ab.err >> gpurun_out/ab.log
done
PW_LIB=paper_2507_17094_b200/libpwb200.so timeout 300 python tools/ab.py --config c2s --tuning '{"row_copy":1}' 2>>gpurun_out/ab.err >> gpurun_out/ab.log
cat gpurun_out/ab.log
