#!/bin/bash
# a2a TMA path on N GPUs: parity suite, C5 sweep with both copy paths, the C2 bench.
out=gpurun_out/${1:-mg4}; N=${2:-4}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_executor.py -q -rA -m gpu -k "mgpu_step or scatter_from or a2a or fused or ring" > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 $N; do for t in 0 1; do
  FSP_A2A_TMA=$t timeout 400 $TR --nproc-per-node $n --master-port $((29780+n+t)) scripts/a2a_sweep.py --max-mb 4096 > $out/sweep_n${n}_tma$t.log 2>&1
done; done
for n in 2 $N; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29720+n)) bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.json 2> $out/bench_n$n.err; echo rc=$? >> $out/bench_n$n.err
done
