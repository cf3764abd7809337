set -x
timeout 300 python tools/profile_h16.py 3 2>&1 | tail -4
PGB_RFI_WIDEN=1 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedisp_h16 -c 1 -o gpurun_out/r3e_h16 python tools/profile_h16.py 1 > gpurun_out/r3e_ncu.log 2>&1; tail -3 gpurun_out/r3e_ncu.log
