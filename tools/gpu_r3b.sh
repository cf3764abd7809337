# fp16 in-order kernel for RFI-masked chunks: parity + config-E timing
set -x
timeout 900 python -m pytest tests/test_gpu_h16.py tests/test_gpu_rfi.py -q -p no:cacheprovider -x > gpurun_out/r3b_pytest.log 2>&1; tail -15 gpurun_out/r3b_pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider -k E1 > gpurun_out/r3b_pytest_e1.log 2>&1; tail -5 gpurun_out/r3b_pytest_e1.log
timeout 900 python tools/bench_configs.py E --steps 2 > gpurun_out/r3b_configE.jsonl 2> gpurun_out/r3b_configE.err; cut -c1-900 gpurun_out/r3b_configE.jsonl; tail -3 gpurun_out/r3b_configE.err
