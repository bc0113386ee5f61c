# TMA tile::gather4 scoring rows (flag 8): parity first (bounded waits), then A/B at the C2 bench point; tail probe
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tma_gather4" > gpurun_out/pytest_tma_r02k.log 2>&1; tail -3 gpurun_out/pytest_tma_r02k.log
timeout 600 python -m pytest tests/test_gpu_u8.py -x -q -m gpu -k "tma" >> gpurun_out/pytest_tma_r02k.log 2>&1; tail -2 gpurun_out/pytest_tma_r02k.log
timeout 1200 python tools/ab.py --config c2 --l 128 --discard 0.75 --ghost-iter 1 --tuning '[{"flags": 2}, {"flags": 10}]' --libs default,tools/lib_t640.so --rounds 2 > gpurun_out/ab_r02k.log 2> gpurun_out/ab_r02k.err; cat gpurun_out/ab_r02k.log; tail -3 gpurun_out/ab_r02k.err
timeout 900 python tools/tail_probe.py --config c2 --l 128 > gpurun_out/tail_c2_r02k.jsonl 2> gpurun_out/tail_c2_r02k.err; cat gpurun_out/tail_c2_r02k.jsonl
