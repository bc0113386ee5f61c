# FAST K1 instances: GPU suite + A/B vs the previous build at the C2 point
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r02aa.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02aa.log
timeout 1500 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs tools/lib_base.so,default --rounds 3 > gpurun_out/ab_fast_r02aa.log 2> gpurun_out/ab_fast_r02aa.err; python -c "
import json
for l in open('gpurun_out/ab_fast_r02aa.log'):
    d=json.loads(l); print(d['lib'], d['round'], 'naive', d['naive']['kernel_ms'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['ids_sum'], d['naive']['ids_sum'])"; tail -2 gpurun_out/ab_fast_r02aa.err
