set -x
timeout 300 python tools/profile_h16.py 3 2>&1 | tail -2
PGB_H16_G=4 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -2
PGB_H16_G=2 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -2
