#!/bin/bash
# Attention length sweep vs cuDNN / flash-attn 2 (one B200): gpurun_out/sweep.log
mkdir -p gpurun_out
for wl in 1024x256 2048x128 4096x64 8192x32 16384x16 32768x8 c2; do
  echo "WL=$wl"; WL=$wl timeout 300 python scripts/perf_attn.py 2>&1 | grep "fwd\|bwd"
done > gpurun_out/sweep.log 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv >> gpurun_out/sweep.log
