timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r02ae.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02ae.log
timeout 1500 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs tools/lib_base.so,default --rounds 3 > gpurun_out/ab_wide_r02ae.log 2> gpurun_out/ab_wide_r02ae.err; python -c "
import json
for l in open('gpurun_out/ab_wide_r02ae.log'):
    d=json.loads(l); print(d['lib'], d['round'], 'naive', d['naive']['kernel_ms'], d['naive']['warps'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['warps'], d['pathweaver']['ids_sum'])"; tail -2 gpurun_out/ab_wide_r02ae.err
