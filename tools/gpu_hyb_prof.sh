# event-replay RFI kernel: launch times on the reduced E chunk and config E1, one ncu capture
set -x
export PG_TEST_ABLATIONS=1 PGB_RFI_HYB=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hyb|dedisp_f32|transpose|rfi|mask" --csv --log-file gpurun_out/hyb_launches.csv python tools/profile_h16.py 2 > gpurun_out/hyb_prof.log 2>&1
python tools/launch_summary.py gpurun_out/hyb_launches.csv | head -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedisp_hyb -c 1 -o gpurun_out/hyb_full python tools/profile_h16.py 1 > gpurun_out/hyb_ncu.log 2>&1
tail -2 gpurun_out/hyb_ncu.log
