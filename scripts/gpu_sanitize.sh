#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over one small step of
# every model (+ the MNIST smoke). Usage: bash scripts/gpu_sanitize.sh [tag]
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 20 python scripts/sanitize_models.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/$tool.log
done
for f in $OUT/*.log; do echo == $f; grep -E "ok|SUMMARY|rc=" $f | tail -8; done
