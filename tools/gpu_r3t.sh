timeout 300 python tools/profile_h16.py 3 2>&1 | tail -1
PGB_RFI_H16=1 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | tail -1
PGB_RFI_H16=1 PGB_H16_NT512=1 PGB_DD_WHICH=1 PG_TEST_ABLATIONS=1 timeout 300 python tools/profile_h16.py 3 2>&1 | grep -v boxcar | tail -3
PGB_RFI_H16=1 PGB_H16_NT512=1 PG_TEST_ABLATIONS=1 timeout 600 python -m pytest tests/test_gpu_h16.py -q -p no:cacheprovider -k "local_mean and True" 2>&1 | tail -2
