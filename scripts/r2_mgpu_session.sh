#!/bin/bash
# Round-2 multi-GPU evidence on one N-GPU box (gpurun --gpus N): parity over real NVSwitch
# (incl. the loader-shard data scatter), cost-model calibration, the bench at N=2/N, and
# the C3 full step with ZeRO-3 vs bf16 replicas.  Outputs under gpurun_out/$1/.
out=gpurun_out/${1:-mg}; N=${2:-4}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
nvidia-smi topo -m > $out/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rA -m gpu -k "mgpu_step or scatter" > $out/pytest_multi.log 2>&1; echo rc=$? >> $out/pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node $N --master-port 29711 scripts/calibrate.py --out $out/calib --per-degree 6 > $out/calib.log 2>&1; echo rc=$? >> $out/calib.log
for n in 2 $N; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29720+n)) bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.json 2> $out/bench_n$n.err; echo rc=$? >> $out/bench_n$n.err
done
timeout 900 $TR --nproc-per-node $N --master-port 29731 bench.py --gpus $N --steps 10 --warmup 3 --impl reference > $out/ref_n$N.json 2>&1
for mode in "" "--replicated"; do
  tag=$([ -z "$mode" ] && echo zero || echo replicated)
  timeout 1500 $TR --nproc-per-node $N --master-port 29741 scripts/bench_full_step.py --steps 2 --warmup 1 $mode > $out/full_$tag.json 2> $out/full_$tag.err; echo rc=$? >> $out/full_$tag.err
done
