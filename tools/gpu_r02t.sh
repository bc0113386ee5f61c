# A/B: DGS parent rows into registers (PW_DGS_LDG) vs staging ring; parity of the variant
timeout 600 env PW_LIB=tools/lib_dgsldg.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "synthetic_matches_oracle or small_golden" > gpurun_out/pytest_dgsldg_r02t.log 2>&1; tail -2 gpurun_out/pytest_dgsldg_r02t.log
timeout 1200 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs default,tools/lib_dgsldg.so --rounds 3 > gpurun_out/ab_r02t.log 2> gpurun_out/ab_r02t.err; python -c "
import json
for l in open('gpurun_out/ab_r02t.log'):
    d=json.loads(l); print(d['lib'], d['round'], 'naive', d['naive']['kernel_ms'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['ids_sum'])"; tail -2 gpurun_out/ab_r02t.err
