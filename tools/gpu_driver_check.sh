# the driver's round-end commands on the current tree
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/dc_bench_default.json 2> gpurun_out/dc_bench_default.err; cut -c1-300 gpurun_out/dc_bench_default.json
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/dc_bench_ref.json 2> gpurun_out/dc_bench_ref.err; cut -c1-500 gpurun_out/dc_bench_ref.json
PG_DIST_BACKEND=gloo PG_SAME_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/dc_bench_2r.json 2> gpurun_out/dc_bench_2r.err; cut -c1-300 gpurun_out/dc_bench_2r.json; tail -3 gpurun_out/dc_bench_2r.err
