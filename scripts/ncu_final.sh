#!/bin/bash
# ncu evidence for the final kernels (one GPU): launch list of a short C2 bench and one
# --set full capture of the attention fwd and bwd launches (profiling recipe of
# /opt/skills/guides/B200_PROFILING.md).  Output in gpurun_out/$1.
out=gpurun_out/${1:-ncufinal}; mkdir -p $out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > $out/plain.json 2> $out/plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv $CMD > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel_v2 -s 2 -c 1 -o $out/bwd $CMD > $out/ncu_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_pair_kernel -s 2 -c 1 -o $out/fwd $CMD > $out/ncu_fwd.log 2>&1
