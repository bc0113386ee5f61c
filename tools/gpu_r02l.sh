# TMA fault repro (sanitizer) + regression A/B across commits
timeout 300 python tools/tma_repro.py 10 64 > gpurun_out/tma_repro_r02l.log 2>&1; tail -2 gpurun_out/tma_repro_r02l.log
timeout 300 python tools/tma_repro.py 8 64 >> gpurun_out/tma_repro_r02l.log 2>&1; tail -2 gpurun_out/tma_repro_r02l.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/tma_repro.py 8 64 > gpurun_out/tma_sanitizer_r02l.log 2>&1; grep -A12 "=====" gpurun_out/tma_sanitizer_r02l.log | head -40
timeout 1200 python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs default,tools/lib_1fb73bd.so,tools/lib_0fef333.so --rounds 2 > gpurun_out/ab_r02l.log 2> gpurun_out/ab_r02l.err; cat gpurun_out/ab_r02l.log | cut -c1-300; tail -3 gpurun_out/ab_r02l.err
