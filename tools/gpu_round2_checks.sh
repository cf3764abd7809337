set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu4.log 2>&1; tail -6 gpurun_out/r2_pytest_gpu4.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err; cut -c1-600 gpurun_out/r2_bench4.json
timeout 600 python tools/shard_timing.py > gpurun_out/r2_shards.jsonl 2>&1; cat gpurun_out/r2_shards.jsonl
timeout 600 python tools/bench_configs.py D Ddisk A --steps 3 > gpurun_out/r2_configsD.jsonl 2> gpurun_out/r2_configsD.err; cut -c1-500 gpurun_out/r2_configsD.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedisp_u8_ring_persist -s 1 -c 1 -o gpurun_out/r2_dd python tools/profile_chunk.py 2 > gpurun_out/r2_ncu_dd.log 2>&1; tail -3 gpurun_out/r2_ncu_dd.log
timeout 600 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_synccheck.log 2>&1; tail -4 gpurun_out/r2_synccheck.log
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_racecheck.log 2>&1; tail -4 gpurun_out/r2_racecheck.log
