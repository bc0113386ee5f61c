# A/B of tools/lib_prev.so vs the working tree (CFG/L/TUNING env) after the parity tests;
# TIMERS=1 adds the per-phase cycle breakdown, NCU=1 an ncu --set full capture of K1.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/ab.log
for i in 1 2; do
PW_LIB=tools/lib_prev.so timeout 900 python tools/ab.py --config ${CFG:-c2} --l ${L:-256} ${TUNING:+--tuning "$TUNING"} 2>>gpurun_out/ab.err >> gpurun_out/ab.log
timeout 900 python tools/ab.py --config ${CFG:-c2} --l ${L:-256} ${TUNING:+--tuning "$TUNING"} 2>>gpurun_out/ab.err >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
if [ -n "$TIMERS" ]; then
python -m paper_2507_17094_b200.build_ext --timers > gpurun_out/build_timers.log 2>&1
PW_LIB=paper_2507_17094_b200/libpwb200_timers.so timeout 900 python tools/phase_timers.py --config ${CFG:-c2} --l ${L:-256} ${TUNING:+--tuning "$TUNING"} > gpurun_out/phase.log 2>>gpurun_out/ab.err
cat gpurun_out/phase.log
fi
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_search -s 2 -c 1 -o gpurun_out/prof_${CFG:-c2}_${TAG:-x} python tools/profile_run.py --config ${CFG:-c2} --l ${L:-256} --reps 3 ${TUNING:+--tuning "$TUNING"} > gpurun_out/prof.log 2>&1
tail -2 gpurun_out/prof.log
fi
