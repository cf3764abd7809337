# round 2, second GPU pass: restructured ring loop, stage timings, drift stress
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_dropin.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; tail -5 gpurun_out/r2b_pytest.log
timeout 300 python tools/dd_variant_timing.py 5 > gpurun_out/r2b_dd.txt 2>&1; cat gpurun_out/r2b_dd.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; cut -c1-400 gpurun_out/r2b_bench.json
timeout 900 python tools/dropin_timing.py --runs 2 > gpurun_out/r2b_dropin.jsonl 2> gpurun_out/r2b_dropin.err; cut -c1-600 gpurun_out/r2b_dropin.jsonl; tail -3 gpurun_out/r2b_dropin.err
