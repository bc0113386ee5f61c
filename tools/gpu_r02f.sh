# bench parity block + choice tail-shuffle GPU test
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tail_shuffle" > gpurun_out/pytest_tail_r02f.log 2>&1; tail -3 gpurun_out/pytest_tail_r02f.log
timeout 600 python bench.py --config tiny --steps 3 > gpurun_out/bench_tiny_r02f.json 2> gpurun_out/bench_tiny_r02f.err; tail -c 1500 gpurun_out/bench_tiny_r02f.json; tail -3 gpurun_out/bench_tiny_r02f.err
timeout 1500 python bench.py > gpurun_out/bench_c2_r02f.json 2> gpurun_out/bench_c2_r02f.err; python -c "import json;d=json.loads(open('gpurun_out/bench_c2_r02f.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e'],d['roofline']['frac'],json.dumps(d['parity']))"; tail -3 gpurun_out/bench_c2_r02f.err
