#!/bin/bash
# counter runs of LAPIS_B200_RS_CHUNK tiles per atomic, by counter share
for DK in "100 5" "100 7" "100 10" "100 12" "100 16" "100 5"; do
  set -- $DK
  echo "== DYN=$1 CHUNK=$2"
  LAPIS_B200_RS_DYN=$1 LAPIS_B200_RS_CHUNK=$2 timeout 300 python scripts/rs_times.py 2>&1 | awk '{print $4, $11, $12, $13, $14, $15}' | tail -6
done
