#!/bin/bash
# Profiling pass run on the GPU box.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
for t in gemm_s8_qkv gemm_s8_o gemm_s8_ff1 gemm_s8_ff2 gemm_s8_8192 gemm_f16_8192 gemm_f16_ff1; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -c 1 \
      -o gpurun_out/prof_$t python tools/prof_targets.py $t 2 > gpurun_out/ncu_$t.log 2>&1
  echo "$t rc=$?"
done
for t in attn_fwd:k_attn_fwd attn_bwd:k_attn_bwd ln_bwd:k_ln_bwd act_bwd:k_act_bwd adamw:k_adamw \
         conv_fwd:k_gemm_tc conv_wgrad:k_gemm_tc conv_dgrad:k_gemm_tc; do
  k=${t#*:}; t=${t%%:*}
  skip=0; [ "$t" = adamw ] && skip=1   # the first k_adamw launch is the weight-prepare pass
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip -c 1 \
      -o gpurun_out/prof_$t python tools/prof_targets.py $t 2 > gpurun_out/ncu_$t.log 2>&1
  echo "$t rc=$?"
done
for t in quantize_with_scale quantize_per_channel absmax stats cast dequantize; do
  timeout 300 ncu --set full --clock-control none -k regex:'k_' -c 1 \
      -o gpurun_out/prof_$t python tools/prof_targets.py $t 1 > gpurun_out/ncu_$t.log 2>&1
  echo "$t rc=$?"
done
