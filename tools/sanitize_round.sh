#!/bin/bash
# compute-sanitizer over tools/sanitize.py: memcheck,
# racecheck and synccheck per kernel group; logs in gpurun_out/sanitize_*.log.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for g in ${SAN_GROUPS:-gemm1 gemm2 conv_tma conv_gather attn1 attn2 sr pdl quant dual streamk gelu1 attnq head}; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $g \
      > gpurun_out/sanitize_${tool}_${g}.log 2>&1
    echo "$tool $g rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${g}.log | tail -1)"
  done
done
