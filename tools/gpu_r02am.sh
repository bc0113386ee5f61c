timeout 1500 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs tools/lib_prev.so,tools/lib_noqreg.so --rounds 3 > gpurun_out/ab_qreg_r02am.log 2> gpurun_out/ab_qreg_r02am.err; python -c "
import json
for l in open('gpurun_out/ab_qreg_r02am.log'):
    d=json.loads(l); print(d['lib'], d['round'], 'naive', d['naive']['kernel_ms'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['ids_sum'], d['naive']['ids_sum'])"; tail -2 gpurun_out/ab_qreg_r02am.err
