timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_multifile.py -q -p no:cacheprovider -x > gpurun_out/stream_pytest.log 2>&1; tail -3 gpurun_out/stream_pytest.log
timeout 800 python tools/fil_timing.py 8 16 > gpurun_out/fil_timing.jsonl 2>&1; grep path gpurun_out/fil_timing.jsonl | cut -c1-300
