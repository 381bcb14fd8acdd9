#!/bin/bash
# Round-end measurement pass on one B200 (outputs in gpurun_out/): GPU tests,
# smoke, bench lines (mixed / int8 / fp16 + reference arm), kernel bench,
# plan step times, CUPTI step trace, then the ncu launch list + captures.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for p in int8 fp16; do timeout 300 python bench.py --plan $p --no-cpu-baseline > gpurun_out/bench_$p.json 2>gpurun_out/bench_$p.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
timeout 900 python bench_kernels.py --json gpurun_out/kbench.json > gpurun_out/kbench.log 2>&1; echo "kbench rc=$?"
timeout 600 python tools/plan_steps.py --json gpurun_out/plan_steps.json > gpurun_out/plan_steps.log 2>&1
timeout 300 python tools/step_trace.py --plan mixed --out gpurun_out/step_trace > /dev/null 2>&1
timeout 300 python tools/gemm_overhead.py > gpurun_out/gemm_overhead.txt 2>&1
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
python tools/summarize_round.py >> gpurun_out/profile_round.log 2>&1
tail -3 gpurun_out/profile_round.log
