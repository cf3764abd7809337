#!/bin/bash
# dedisp timing sweep over staging geometries (experiments)
for cfg in "8 3" "4 6" "4 4" "2 8"; do
  set -- $cfg
  PGB_DD_WS=1 PGB_WS_G=$1 PGB_WS_NS=$2 timeout 120 python tools/profile_chunk.py 2 2>&1 | sed "s/^/G=$1 NS=$2 /"
done
timeout 120 python tools/profile_chunk.py 2 2>&1 | sed "s/^/classic /"
