set -x
timeout 900 python -m pytest tests/test_gpu_h16.py tests/test_gpu_rfi.py tests/test_gpu_configs.py -q -p no:cacheprovider -k "not config_file or E1" > gpurun_out/r3i_pytest.log 2>&1; tail -5 gpurun_out/r3i_pytest.log
timeout 900 python tools/bench_configs.py E --steps 2 > gpurun_out/r3i_configE.jsonl 2> gpurun_out/r3i_configE.err; cut -c1-400 gpurun_out/r3i_configE.jsonl
