#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of one implicit step (C1,
# C2 kappa=1e6) through the public API; summaries into gpurun_out/sanitize/.
cd "$(dirname "$0")/.."
out=gpurun_out/sanitize
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in ${CFGS:-C1 C2}; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report hazard"
    timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 50 \
      python tools/sanitize_step.py $cfg > $out/${cfg}_${tool}.log 2>&1
    echo "$cfg $tool rc=$?" | tee -a $out/summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" $out/${cfg}_${tool}.log | tail -5 >> $out/summary.txt
  done
done
