timeout 300 python tools/dd_variant_timing.py 4 2>&1 | tail -1
PGB_DD_2CTA=1 PGB_DD_WHICH=1 timeout 300 python tools/dd_variant_timing.py 4 2>&1 | tail -2
