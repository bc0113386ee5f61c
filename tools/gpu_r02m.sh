# TMA alignment fix + regression A/B (cfg index, original issue sites, TMA compiled out)
timeout 300 python tools/tma_repro.py 8 64 > gpurun_out/tma_repro_r02m.log 2>&1; tail -1 gpurun_out/tma_repro_r02m.log
timeout 300 python tools/tma_repro.py 10 600 >> gpurun_out/tma_repro_r02m.log 2>&1; tail -1 gpurun_out/tma_repro_r02m.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_u8.py -x -q -m gpu -k "tma" > gpurun_out/pytest_tma_r02m.log 2>&1; tail -2 gpurun_out/pytest_tma_r02m.log
timeout 1200 python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '[{"flags": 2}, {"flags": 10}]' --libs default,tools/lib_notma.so,tools/lib_1fb73bd.so --rounds 2 > gpurun_out/ab_r02m.log 2> gpurun_out/ab_r02m.err; cut -c1-330 gpurun_out/ab_r02m.log; tail -3 gpurun_out/ab_r02m.err
