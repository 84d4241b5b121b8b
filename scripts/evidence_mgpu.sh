#!/bin/bash
# Round-end multi-GPU evidence (gpurun --gpus 4, repo root): C2 bench lines at N=2 and 4,
# C3 / C4 attention-layer lines at N=4.
set -u
O=gpurun_out/ev
mkdir -p $O
run() {  # n port args...
  local n=$1 port=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@"
}
run 2 29612 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$?
run 4 29614 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$?
run 4 29615 --config c3 --no-e2e --no-planner > $O/bench_c3_n4.json 2> $O/bench_c3_n4.err; echo c3=$?
run 4 29616 --config c4 --no-e2e --no-planner > $O/bench_c4_n4.json 2> $O/bench_c4_n4.err; echo c4=$?
