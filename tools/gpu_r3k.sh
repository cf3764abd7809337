set -x
timeout 900 python -m pytest tests/test_gpu_boxcar.py tests/test_gpu_parity.py tests/test_gpu_limits.py -q -p no:cacheprovider -x > gpurun_out/r3k_pytest.log 2>&1; tail -15 gpurun_out/r3k_pytest.log
PGB_TRACE=1 timeout 600 python tools/profile_file.py 1 0 2 > gpurun_out/r3k_trace.log 2>&1; grep -E "boxcar|dedisp|chunks done|link" gpurun_out/r3k_trace.log | tail -16
