#!/bin/bash
# dev tool: run the quick checks under several plan overrides, labelled
for mode in "" "FBF_NO_TMA=1" "FBF_BLOCKS_PER_SM=1" "FBF_NO_TMA=1 FBF_BLOCKS_PER_SM=1"; do
  echo "=== mode: [$mode]"
  env $mode timeout 300 python tools/gpu_check.py > gpurun_out/check.log 2>&1; echo "rc=$?"; grep -E "worst|c1:|Error|error" gpurun_out/check.log | head -3
done
