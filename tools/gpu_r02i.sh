# extension knobs: GPU tests vs oracle, then the logical-shard projection with the knobs
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r02i.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02i.log
timeout 2400 python tools/logical_ring.py --config c2 --ns 2,4,8 --ext --pw-grid 0.75:1,0.8:1 > gpurun_out/logical_ext_r02i.jsonl 2> gpurun_out/logical_ext_r02i.err; cat gpurun_out/logical_ext_r02i.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_shards'], d['naive'], d['pathweaver'], d.get('pw_over_naive'), d.get('extension_best'), d.get('ext_over_naive'))"; tail -3 gpurun_out/logical_ext_r02i.err
