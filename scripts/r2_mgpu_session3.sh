#!/bin/bash
# Round-2 final multi-GPU checks (gpurun --gpus N): the full multi-GPU parity suite on real
# NVSwitch and the C3 full step with ZeRO-3 (AdamW) vs replicas.  Outputs under gpurun_out/$1/.
out=gpurun_out/${1:-mg3}; N=${2:-4}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_executor.py -q -rA -m gpu > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for mode in "--optimizer adamw" "--replicated"; do
  tag=$(echo $mode | tr -d ' -')
  timeout 1500 $TR --nproc-per-node $N --master-port 29741 scripts/bench_full_step.py --steps 2 --warmup 1 $mode > $out/full_$tag.json 2> $out/full_$tag.err; echo rc=$? >> $out/full_$tag.err
done
