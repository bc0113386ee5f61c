# e2e: K1 launched before the rest of the query upload, error flags read with the results;
# device value: one-rank batches enqueued without host sync
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_aq.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "upload or pw_run or run_host or smoke or golden or acceptance or streamed" > gpurun_out/pytest_aq.log 2>&1; tail -2 gpurun_out/pytest_aq.log
timeout 1500 python tools/e2e_ab.py --config c2 --libs tools/lib_e2e0.so,default+nostream,default --steps 30 --rounds 3 > gpurun_out/e2e_ab_r02aq.jsonl 2> gpurun_out/e2e_ab_r02aq.err
python -c "
import json
for l in open('gpurun_out/e2e_ab_r02aq.jsonl'):
    d=json.loads(l); print(d['lib'], d['round'], d['ms_per_call'], d['e2e_qps'], d['recall'], d.get('call_us'))
    tl=d.get("timeline", []); [print("   ", t) for t in tl if t[2]=="kernel" or t[0] > 1000]
"
