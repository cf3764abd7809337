# round-2 (session 3) evidence: full gpu suite, bench line, per-config lines, launch list,
# ncu captures of the dominant kernel and the boxcar, memcheck on the new kernels
set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3r_pytest_gpu.log 2>&1; tail -4 gpurun_out/r3r_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r3r_bench.json 2> gpurun_out/r3r_bench.err; cut -c1-400 gpurun_out/r3r_bench.json
timeout 1200 python tools/bench_configs.py A --steps 100 > gpurun_out/r3r_configs.jsonl 2> gpurun_out/r3r_configs.err
timeout 1200 python tools/bench_configs.py C E --steps 2 >> gpurun_out/r3r_configs.jsonl 2>> gpurun_out/r3r_configs.err
timeout 1200 python tools/bench_configs.py D Ddisk --steps 3 >> gpurun_out/r3r_configs.jsonl 2>> gpurun_out/r3r_configs.err
cut -c1-300 gpurun_out/r3r_configs.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r3r_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r3r_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedisp_u8_ring_persist -c 1 -o gpurun_out/r3r_dd python tools/profile_chunk.py 1 > gpurun_out/r3r_ncu_dd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:boxcar_prefix -c 1 -o gpurun_out/r3r_bx python tools/profile_chunk.py 1 > gpurun_out/r3r_ncu_bx.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_boxcar.py tests/test_gpu_h16.py -q -p no:cacheprovider -k "spike_tiles_match or integer_masks or local_mean" > gpurun_out/r3r_memcheck.log 2>&1; tail -5 gpurun_out/r3r_memcheck.log
