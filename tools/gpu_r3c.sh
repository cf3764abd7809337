set -x
PGB_DD_WHICH=1 PGB_TRACE=1 timeout 600 python tools/e1_which.py > gpurun_out/r3c_e1.log 2>&1; grep -v "^\[pgb trace\]" gpurun_out/r3c_e1.log | tail -20; grep "pgb trace" gpurun_out/r3c_e1.log | tail -30
timeout 900 python -m pytest tests/test_gpu_h16.py -q -p no:cacheprovider > gpurun_out/r3c_pytest.log 2>&1; tail -15 gpurun_out/r3c_pytest.log
