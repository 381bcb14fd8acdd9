set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -5 gpurun_out/gputest.log
timeout 900 python bench_kernels.py --sweep --json gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
for t in quantize_with_scale:k_quantize quantize_f16:k_quantize quantize_per_channel:k_quant_rows quantize_per_tensor:k_quantize absmax:k_absmax; do
  k=${t#*:}; t=${t%%:*}
  timeout 300 ncu --set full --clock-control none -k regex:$k -c 1 -o gpurun_out/prof_$t python tools/prof_targets.py $t 1 > gpurun_out/ncu_$t.log 2>&1
  echo "$t rc=$?"
done
python tools/summarize_round.py
