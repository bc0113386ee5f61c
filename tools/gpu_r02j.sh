# tail of the persistent K1 at the C2 bench point (K1 time vs batch size), 16 vs 20 warps/SM
timeout 900 python tools/tail_probe.py --config c2 --l 128 > gpurun_out/tail_c2_r02j.jsonl 2> gpurun_out/tail_c2_r02j.err; cat gpurun_out/tail_c2_r02j.jsonl
timeout 900 python tools/tail_probe.py --config c2 --l 128 --tuning '{"flags": 2, "warps_per_sm": 12}' > gpurun_out/tail_c2_w12_r02j.jsonl 2>&1; cat gpurun_out/tail_c2_w12_r02j.jsonl | grep arm
