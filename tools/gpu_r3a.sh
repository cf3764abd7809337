# re-establish: gpu tests + bench line on the restored tree
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3a_pytest_gpu.log 2>&1; tail -6 gpurun_out/r3a_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; cut -c1-1500 gpurun_out/r3a_bench.json; tail -3 gpurun_out/r3a_bench.err
