#!/bin/bash
# Plan fuzzing on one GPU: random long-tail batches planned by the reference planner at run
# time (tests/vrank_parity.py fuzz<SEED>_n<WORLD>), executed on WORLD virtual ranks and
# checked densely against the CPU oracle.   bash scripts/fuzz_vranks.sh FIRST LAST > log
export CUDA_DEVICE_MAX_CONNECTIONS=32 CUDA_MODULE_LOADING=EAGER FSP_BARRIER_TIMEOUT_S=60 OMP_NUM_THREADS=4
heads=(5 6 7 8 9 10 12 13 16)
pass=0; fail=0; rej=0; inf=0
for s in $(seq $1 $2); do
  w=$(( s % 3 == 0 ? 2 : (s % 3 == 1 ? 4 : 8) )); h=${heads[$(( s % ${#heads[@]} ))]}; d=$(( s % 5 == 0 ? 64 : 128 ))
  out=$(timeout 300 python tests/vrank_parity.py dense fuzz${s}_n$w $w $h $d 2>&1)
  rc=$?
  plan=$(echo "$out" | grep '^{"fuzz"' | head -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read() or "{}"); print(d.get("degrees"), len(d.get("lengths", [])), sum(d.get("lengths", [])))' 2>/dev/null)
  if [ $rc -eq 0 ] && echo "$out" | grep -q '"ok": true'; then pass=$((pass+1)); st=ok
  elif echo "$out" | grep -q "heads cannot be split over SP degree"; then
    rej=$((rej+1)); st="rejected as it must be (fewer heads than the plan's SP degree: LayoutError)"
  elif echo "$out" | grep -q "seqplan.domain.InfeasibleError"; then
    inf=$((inf+1)); st="no plan: the reference planner reports the instance infeasible"
  else fail=$((fail+1)); st="FAIL rc=$rc"; fi
  echo "seed $s world $w heads $h head_dim $d groups $plan: $st"
  case "$st" in FAIL*) echo "$out" | tail -5;; esac
done
echo "passed $pass rejected $rej infeasible $inf failed $fail"
