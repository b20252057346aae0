#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_run.py: racecheck, synccheck and
# memcheck on every kernel family (reduced shapes).  Output -> gpurun_out/.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  for part in ${PARTS:-grid4 general list stage quantile head front5}; do
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_run.py $part \
      > gpurun_out/sanitize_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${part}.txt | tail -1)"
  done
done
