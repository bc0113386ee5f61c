# A/B: resident warps with the FAST K1 (16 default, 20, 24)
timeout 1500 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs default,tools/lib_t640.so,tools/lib_t768.so --rounds 3 > gpurun_out/ab_warps_r02ad.log 2> gpurun_out/ab_warps_r02ad.err; python -c "
import json
for l in open('gpurun_out/ab_warps_r02ad.log'):
    d=json.loads(l); print(d['lib'], d['round'], 'naive', d['naive']['kernel_ms'], d['naive']['warps'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['warps'], d['pathweaver']['smem'], d['pathweaver']['ids_sum'])"; tail -2 gpurun_out/ab_warps_r02ad.err
