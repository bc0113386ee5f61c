# geometric upload chunks: upload tests + e2e A/B (with one GPU timeline per library) vs the previous build
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "upload or result_block or one_shard" > gpurun_out/pytest_upload_s9.log 2>&1; tail -2 gpurun_out/pytest_upload_s9.log
timeout 1200 python tools/e2e_ab.py --config c2 --l 112 --discard 0.75 --ghost-iter 1 --libs tools/lib_prev.so,default --steps 20 --rounds 3 > gpurun_out/e2e_ab_s9.jsonl 2> gpurun_out/e2e_ab_s9.err; cut -c1-200 gpurun_out/e2e_ab_s9.jsonl
