# dedispersion variant timing: 1024-thread ring vs the 512-thread default (ablation library)
set -x
timeout 600 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider > gpurun_out/r2c_variants.log 2>&1; tail -3 gpurun_out/r2c_variants.log
for e in "PGB_RING_MODE=8" "PGB_DD_WARPS=32" "PGB_RING_MODE=8" "PGB_DD_WARPS=32"; do env $e timeout 300 python tools/dd_variant_timing.py 5; done > gpurun_out/r2c_dd.txt 2>&1; cat gpurun_out/r2c_dd.txt
