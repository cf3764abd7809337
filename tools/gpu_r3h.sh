timeout 300 python tools/profile_h16.py 3 2>&1 | tail -1
PGB_H16_UNROLL=1 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -1
PGB_H16_UNROLL=8 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -1
PGB_RFI_WIDEN=1 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -1
