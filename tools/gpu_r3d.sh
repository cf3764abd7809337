set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedisp_h16 -c 1 -o gpurun_out/r3d_h16 python tools/e1_which.py > gpurun_out/r3d_ncu.log 2>&1; tail -3 gpurun_out/r3d_ncu.log
