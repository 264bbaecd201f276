#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over a small set of GPU
# parity tests (ragged tails, swizzled layout, formats, batched launches,
# row-fused per-row G, fused amax, the FP32 block routine).
mkdir -p gpurun_out
SEL='test_parity_small and 129 or test_empty_and_tiny or test_parity_adversarial or test_batched_matches_oracle or test_swizzled_scales or test_format_adversarial or test_tensor_amax_batched or test_dequantize or test_row_fused_batched_mixed or test_row_fused_unit_split or test_row_fused_swizzled or test_fused_corner_tensors or test_fused_nonfinite_flag or test_fused_repeated or (test_fused_equals_separate and window0) or (test_f32_equals_bf16_path and gaussian) or test_f32_nonfinite or test_cuda_graph_tensor_mode or test_small_path_sums or test_next_amax_call or (test_gen_parity and (e2m1_ue4m3_b16 or e3m0_ue4m3_b16 or e2m1_ue8m0_b32)) or test_gen_device_amax or test_peer_exchange_world1'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_parity_gpu.py tests/test_nvfp4_layouts_gpu.py tests/test_formats_gpu.py tests/test_row_fused_gpu.py \
    tests/test_fused_amax_gpu.py tests/test_device_routine_gpu.py tests/test_small_path_gpu.py \
    tests/test_gen_gpu.py tests/test_dist_gpu.py \
    -m gpu -q -x -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
