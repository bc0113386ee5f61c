# A/B: resident query-warps per SM (16 default, 20, 22) at the C2 bench point
timeout 1200 python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs default,tools/lib_t640.so,tools/lib_t704.so --rounds 2 > gpurun_out/ab_r02h.log 2> gpurun_out/ab_r02h.err; cat gpurun_out/ab_r02h.log; tail -3 gpurun_out/ab_r02h.err
