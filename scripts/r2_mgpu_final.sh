#!/bin/bash
# End-of-round confirmation on N GPUs of one box: the whole GPU suite (multi-GPU cases on
# real NVSwitch), then the C2 bench and reference arm at N=2 and N, as the driver launches them.
out=gpurun_out/${1:-mgfinal}; N=${2:-4}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
S=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q -rfE > $out/pytest.log 2>&1; echo "rc=$? secs=$(( $(date +%s) - S ))" >> $out/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 $N; do
  timeout 900 $TR --nproc-per-node $n --master-port $((29720+n)) bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.json 2> $out/bench_n$n.err; echo rc=$? >> $out/bench_n$n.err
  timeout 600 $TR --nproc-per-node $n --master-port $((29740+n)) bench.py --impl reference --gpus $n --steps 3 --warmup 1 > $out/ref_n$n.json 2>> $out/bench_n$n.err
done
