# chunk flags by stream memory op vs by 4-byte copies (PW_UPLOAD_FLAG=copy): upload tests + e2e A/B; 2-rank bench (gloo plumbing default)
set -x
PW_UPLOAD_FLAG=copy timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "upload or result_block or one_shard" > gpurun_out/pytest_upload_s10.log 2>&1; tail -2 gpurun_out/pytest_upload_s10.log
for r in 1 2; do
timeout 600 python tools/e2e_ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --libs default --steps 20 --rounds 2 > gpurun_out/e2e_flagop_s10_$r.jsonl 2>/dev/null; cut -c1-120 gpurun_out/e2e_flagop_s10_$r.jsonl
PW_UPLOAD_FLAG=copy timeout 600 python tools/e2e_ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --libs default --steps 20 --rounds 2 > gpurun_out/e2e_flagcopy_s10_$r.jsonl 2>/dev/null; cut -c1-120 gpurun_out/e2e_flagcopy_s10_$r.jsonl
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --config c2s --no-cpu > gpurun_out/bench_c2s_2ranks_s10.json 2> gpurun_out/bench_c2s_2ranks_s10.err; tail -c 600 gpurun_out/bench_c2s_2ranks_s10.json
