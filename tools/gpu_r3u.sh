timeout 900 python -m pytest tests/test_gpu_boxcar.py tests/test_gpu_parity.py tests/test_gpu_limits.py tests/test_gpu_h16.py -q -p no:cacheprovider -x > gpurun_out/r3u_pytest.log 2>&1; tail -3 gpurun_out/r3u_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:boxcar --csv python tools/profile_chunk.py 1 2>/dev/null | grep -i boxcar | awk -F'","' '{print $5, $NF}' | cut -c1-50,200-260
PGB_TRACE=1 timeout 600 python tools/profile_file.py 1 0 2 > gpurun_out/r3u_trace.log 2>&1; grep -E "chunks done|link" gpurun_out/r3u_trace.log | tail -2
