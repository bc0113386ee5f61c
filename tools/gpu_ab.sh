# A/B of tools/lib_prev.so vs the working tree at C2 (l=256) after the parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/ab.log
for i in 1 2; do
PW_LIB=tools/lib_prev.so timeout 900 python tools/ab.py --config ${CFG:-c2} --l ${L:-256} 2>>gpurun_out/ab.err >> gpurun_out/ab.log
timeout 900 python tools/ab.py --config ${CFG:-c2} --l ${L:-256} ${TUNING:+--tuning "$TUNING"} 2>>gpurun_out/ab.err >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
if [ -n "$TIMERS" ]; then
python -m paper_2507_17094_b200.build_ext --timers > gpurun_out/build_timers.log 2>&1
PW_LIB=paper_2507_17094_b200/libpwb200_timers.so timeout 900 python tools/phase_timers.py --config ${CFG:-c2} --l ${L:-256} > gpurun_out/phase.log 2>>gpurun_out/ab.err
cat gpurun_out/phase.log
fi
