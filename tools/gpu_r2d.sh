# per-config lines with clocks; multi-rank bench path on one GPU (gloo, shared device)
set -x
timeout 900 python tools/bench_configs.py A --steps 200 > gpurun_out/r2d_configs.jsonl 2> gpurun_out/r2d_configs.err
timeout 900 python tools/bench_configs.py C E --steps 2 >> gpurun_out/r2d_configs.jsonl 2>> gpurun_out/r2d_configs.err
timeout 900 python tools/bench_configs.py D Ddisk --steps 5 >> gpurun_out/r2d_configs.jsonl 2>> gpurun_out/r2d_configs.err
cut -c1-700 gpurun_out/r2d_configs.jsonl; tail -3 gpurun_out/r2d_configs.err
PG_DIST_BACKEND=gloo PG_SAME_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_2ranks_gloo.json 2> gpurun_out/r2d_bench_2ranks_gloo.err; cut -c1-900 gpurun_out/r2d_bench_2ranks_gloo.json; tail -5 gpurun_out/r2d_bench_2ranks_gloo.err
