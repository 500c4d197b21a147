#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family of libslip on
# small shapes: pair and non-pair GEMMs (every epilogue incl. the fused B-pass
# reductions), the grouped / merged W launch, attention fwd / dQ / dK-dV, LayerNorm fwd /
# bwd, column reductions + finalize, MSE, AdamW (+ rollback), synthetic inputs, and the
# N = 1 executor.  Logs: gpurun_out/sanitize_<tool>.log (summary line at the end of each).
#   bash tools/sanitize.sh            (on the GPU box, from the repo root)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
TESTS=(
  "tests/test_gpu_stage.py::test_stage_step_matches_oracle[c1]"
  "tests/test_gpu_stage.py::test_stage_step_matches_oracle[d80_ragged]"
  "tests/test_gpu_stage.py::test_weight_multi_matches_oracle[d80_ragged]"
  "tests/test_gpu_stage.py::test_adamw_matches_oracle"
  "tests/test_gpu_stage.py::test_adamw_rollback_reverses_the_step"
  "tests/test_gpu_stage.py::test_mse_head_and_synth"
  "tests/test_gpu_gemm.py"
  "tests/test_gpu_attention.py::test_attention_fwd_bwd_vs_torch[200-3-2-128-1.0]"
  "tests/test_gpu_attention.py::test_attention_fwd_bwd_vs_torch[300-2-1-80-1.0]"
  "tests/test_gpu_attention.py::test_attention_fwd_bwd_vs_torch[96-2-1-32-1.0]"
  "tests/test_gpu_executor.py::test_execute_schedule_n1_matches_oracle[c1]"
)
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitize_$tool.log
  : > $log
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  for t in "${TESTS[@]}"; do
    echo "=== $tool $t" >> $log
    timeout 900 $CS --tool $tool $extra --error-exitcode 99 --print-limit 20 \
      python -m pytest -q -p no:cacheprovider "$t" >> $log 2>&1
    echo "rc=$? ($tool $t)" >> $log
  done
done
grep -h "^rc=\|ERROR SUMMARY" gpurun_out/sanitize_*.log > gpurun_out/sanitize_summary.txt
