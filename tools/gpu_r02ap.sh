# e2e: K1 launched before the rest of the query upload, error flags read with the results;
# device value: one-rank batches enqueued without host sync
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ap.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "upload or pw_run or run_host or smoke" > gpurun_out/pytest_ap.log 2>&1; tail -2 gpurun_out/pytest_ap.log
timeout 1500 python tools/e2e_ab.py --config c2 --libs tools/lib_e2e0.so,default --steps 20 --rounds 2 > gpurun_out/e2e_ab_r02ap.jsonl 2> gpurun_out/e2e_ab_r02ap.err
python -c "
import json
for l in open('gpurun_out/e2e_ab_r02ap.jsonl'):
    d=json.loads(l); print(d['lib'], d['round'], d['ms_per_call'], d['e2e_qps'], d['recall'], d.get('call_us'))
    for t in d.get('timeline', []): print('   ', t)
"
