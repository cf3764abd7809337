# round-2 evidence (session 4): full gpu suite, bench line, per-config lines, launch list,
# ncu captures of the dedispersion ring and the boxcar, sanitizer
set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev3_pytest_gpu.log 2>&1; tail -4 gpurun_out/ev3_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/ev3_bench.json 2> gpurun_out/ev3_bench.err; cut -c1-400 gpurun_out/ev3_bench.json
timeout 1200 python tools/bench_configs.py A --steps 100 > gpurun_out/ev3_configs.jsonl 2> gpurun_out/ev3_configs.err
timeout 1200 python tools/bench_configs.py C E E1 E1norfi --steps 2 >> gpurun_out/ev3_configs.jsonl 2>> gpurun_out/ev3_configs.err
timeout 1200 python tools/bench_configs.py D Ddisk --steps 3 >> gpurun_out/ev3_configs.jsonl 2>> gpurun_out/ev3_configs.err
cut -c1-300 gpurun_out/ev3_configs.jsonl
timeout 900 python tools/fil_timing.py 8 > gpurun_out/ev3_fil_timing.jsonl 2>&1; grep path gpurun_out/ev3_fil_timing.jsonl | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev3_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev3_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedisp_u8_ring_persist -c 1 -o gpurun_out/ev3_dd python tools/profile_chunk.py 1 > gpurun_out/ev3_ncu_dd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:boxcar_prefix -c 1 -o gpurun_out/ev3_bx python tools/profile_chunk.py 1 > gpurun_out/ev3_ncu_bx.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_stream.py tests/test_gpu_boxcar.py -q -p no:cacheprovider -k "pieces or unreadable or spike_tiles_match" > gpurun_out/ev3_memcheck.log 2>&1; tail -3 gpurun_out/ev3_memcheck.log
