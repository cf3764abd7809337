timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_limits.py -q -p no:cacheprovider -x -k "not C1 and not E1" > gpurun_out/r3s_pytest.log 2>&1; tail -2 gpurun_out/r3s_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:baseline --csv python tools/profile_chunk.py 1 2>/dev/null | grep -i baseline | awk -F'","' '{print $5, $NF}' | cut -c1-50,200-260
PGB_TRACE=1 timeout 600 python tools/profile_file.py 1 0 2 > gpurun_out/r3s_trace.log 2>&1; grep -E "chunks done|link" gpurun_out/r3s_trace.log | tail -2
