#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root): smoke, GPU tests,
# the N=1 bench line, the reference arm, the ncu launch list of the bench and one
# `ncu --set full` capture each of the attention backward / forward main kernels.
set -u
O=gpurun_out/ev
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $O/pytest_gpu.log
timeout 500 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo bench=$?
timeout 500 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err; echo ref=$?
FAST="--no-static --no-cpu --no-planner --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 $FAST > $O/ncu_launches.log 2>&1; echo launches=$?
for k in attn_bwd_kernel_v2 attn_fwd_pair_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 3 -c 1 \
    -o $O/prof_$k python bench.py --steps 1 --warmup 3 $FAST > $O/ncu_$k.log 2>&1; echo ncu_$k=$?
  ncu -i $O/prof_$k.ncu-rep --page raw --csv > $O/raw_$k.csv 2>/dev/null
  ncu -i $O/prof_$k.ncu-rep --page details --csv > $O/details_$k.csv 2>/dev/null
  ls -la $O/prof_$k.ncu-rep
done
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt; nproc >> $O/gpu.txt
