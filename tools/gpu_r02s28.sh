# final tree: C5s and c2h lines
set -x
timeout 1800 python bench.py --config c5s > gpurun_out/bench_c5s_s28.json 2> gpurun_out/bench_c5s_s28.err; tail -c 200 gpurun_out/bench_c5s_s28.json
timeout 1800 python bench.py --config c2h > gpurun_out/bench_c2h_s28.json 2> gpurun_out/bench_c2h_s28.err; tail -c 200 gpurun_out/bench_c2h_s28.json
