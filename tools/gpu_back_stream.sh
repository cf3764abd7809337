# back halves on their own stream: A/B timing, full gpu suite, bench, memcheck of file searches
set -x
timeout 900 python tools/back_stream_ab.py B A C1 E1 2>&1 | tail -5 > gpurun_out/bs_ab.jsonl; cat gpurun_out/bs_ab.jsonl
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bs_pytest_gpu.log 2>&1; tail -4 gpurun_out/bs_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bs_bench.json 2> gpurun_out/bs_bench.err; cut -c1-400 gpurun_out/bs_bench.json
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_h16.py -q -p no:cacheprovider -k "h16_equals_float" > gpurun_out/bs_memcheck.log 2>&1; tail -3 gpurun_out/bs_memcheck.log
