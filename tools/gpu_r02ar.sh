# chunked upload enqueued before the launch again (ncu / CUDA_LAUNCH_BLOCKING safe); launch list of the bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ar.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "upload or pw_run or one_shard or blocking" > gpurun_out/pytest_ar.log 2>&1; tail -2 gpurun_out/pytest_ar.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_search|reduce_topk|fill|gather_rows|init_run" --csv --log-file gpurun_out/launches_c2_final3.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu_final3.log 2>&1; tail -c 300 gpurun_out/bench_ncu_final3.log
timeout 1500 python tools/e2e_ab.py --config c2 --libs tools/lib_e2e0.so,default --steps 30 --rounds 3 > gpurun_out/e2e_ab_r02ar.jsonl 2> gpurun_out/e2e_ab_r02ar.err
python -c "
import json
for l in open('gpurun_out/e2e_ab_r02ar.jsonl'):
    d=json.loads(l); print(d['lib'], d['round'], d['ms_per_call'], d['e2e_qps'], d['recall'], d.get('call_us'))
"
