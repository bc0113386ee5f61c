# A/B: FAST launches clear only the dedup hash's key half, once per iteration
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_as.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dataflow.py tests/test_gpu_u8.py tests/test_gpu_ip.py -q -m gpu -x > gpurun_out/pytest_gpu_r02as.log 2>&1; tail -2 gpurun_out/pytest_gpu_r02as.log
timeout 1500 python tools/ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --tuning '{"flags": 2}' --libs tools/lib_e2e0.so,default --rounds 5 > gpurun_out/ab_bh_r02as.log 2> gpurun_out/ab_bh_r02as.err; python -c "
import json
for l in open('gpurun_out/ab_bh_r02as.log'):
    d=json.loads(l); print(d['lib'], d['round'], 'naive', d['naive']['kernel_ms'], 'pw', d['pathweaver']['kernel_ms'], d['pathweaver']['ids_sum'], d['naive']['ids_sum'])"; tail -2 gpurun_out/ab_bh_r02as.err
