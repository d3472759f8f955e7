#!/bin/bash
# compute-sanitizer over a representative subset of the GPU kernel tests
# (memcheck / racecheck / synccheck).  Under the sanitizer every
# kernel runs serialised and instrumented (10-100x slower), so the subset is
# the small-shape parity tests: aggregation fwd/bwd (scalar, float4, slab,
# u8 argmax), force head, batch assembly (fused + multi-kernel), loss /
# Adam / guard, the tcgen05 GEMM engine (through the C1 model and small
# cases), ragged capacity batches, the store-mode gather and the EGNN kernels.
# Usage (under gpurun): tools/sanitize.sh  -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SEL="test_aggregate_fwd_bwd_bitwise_fp64 or test_aggregate_fp32_vectorised_vs_oracle or test_force_head_fp32_wide or test_fused_radius_batch or test_c1_model_fp32 or test_small_cases_vs_reference_golden or test_trainer_step_fp64 or test_guard_advance or test_egnn_vs_oracle or test_ragged_runner_matches_oracle or test_store_gather_batch or test_deferred_batched"
export GFM_NO_PDL=1  # plain launches: the sanitizer serialises kernels anyway
for tool in memcheck racecheck synccheck; do
  timeout 3000 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "$SEL" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_summary.log
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.log
done
