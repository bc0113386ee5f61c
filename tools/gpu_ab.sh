# A/B of several libraries (LIBS, default "tools/lib_prev.so default") at CFG/L/TUNING after
# the parity tests; TIMERS=1 adds the per-phase cycle breakdown, NCU=1 an ncu capture of K1.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; fi
: > gpurun_out/ab.log
for i in 1 2; do
for lib in ${LIBS:-tools/lib_prev.so default}; do
  if [ "$lib" = default ]; then unset PW_LIB; else export PW_LIB=$lib; fi
  timeout 900 python tools/ab.py --config ${CFG:-c2} --l ${L:-256} ${TUNING:+--tuning "$TUNING"} 2>>gpurun_out/ab.err >> gpurun_out/ab.log
done
done
unset PW_LIB
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
