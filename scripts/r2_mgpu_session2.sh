#!/bin/bash
# Round-2 multi-GPU session 2 (gpurun --gpus N): parity of the persistent fused-scatter
# attention and of ring attention over real NVSwitch, the C2/C3/C4 bench lines at N=2/N,
# and context-parallel timings of one long sequence.  Outputs under gpurun_out/$1/.
out=gpurun_out/${1:-mg2}; N=${2:-4}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rA -m gpu -k "mgpu_step or ring or scatter_from" > $out/pytest_multi.log 2>&1; echo rc=$? >> $out/pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 $N; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29720+n)) bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.json 2> $out/bench_n$n.err; echo rc=$? >> $out/bench_n$n.err
done
for cfg in c3 c4; do
  timeout 1200 $TR --nproc-per-node $N --master-port 29735 bench.py --gpus $N --steps 5 --warmup 3 --config $cfg --no-e2e --no-cpu > $out/bench_${cfg}_n$N.json 2> $out/bench_${cfg}_n$N.err; echo rc=$? >> $out/bench_${cfg}_n$N.err
done
for S in 393216 1048576; do
  timeout 900 $TR --nproc-per-node $N --master-port 29745 scripts/ring_parity.py $S 8 --no-check > $out/ring_$S.json 2> $out/ring_$S.err; echo rc=$? >> $out/ring_$S.err
done
