#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize.py
OUT=gpurun_out/${1:-sanitize}; mkdir -p $OUT
for T in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize.py ${CASES} > $OUT/sanitizer_$T.txt 2>&1
  echo "$T rc=$?"; tail -4 $OUT/sanitizer_$T.txt
done
