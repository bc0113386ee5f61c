# early K1 launch (chunk 0 ahead, the rest behind; gated on launches that may block): upload tests, e2e A/B, e2e with PW_UPLOAD_ALL_FIRST
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "upload or result_block or one_shard" > gpurun_out/pytest_upload_s14.log 2>&1; tail -2 gpurun_out/pytest_upload_s14.log
timeout 900 python tools/e2e_ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --libs tools/lib_prev.so,default --steps 20 --rounds 3 > gpurun_out/e2e_ab_s14.jsonl 2> gpurun_out/e2e_ab_s14.err; cut -c1-150 gpurun_out/e2e_ab_s14.jsonl
