# A/B of backward-kernel build knobs against the default build. Variants are built with
# scripts/build_variant.sh NAME -D...; run as: bash scripts/ab_bwd_knobs.sh NAME [NAME ...]
# (round 1: ring4 -DFSP_BWD_RING=4, cw8 -DFSP_BWD_COMPUTE_WARPS=8 when 16 was the default,
# cw4 -DFSP_BWD_COMPUTE_WARPS=4, red8 -DFSP_BWD_REDUCE_WARPS=8). Parity, then C2 / 32K timings.
mkdir -p gpurun_out/abb
for v in "$@"; do
  FSP_LIB=paper_2412_01523_b200/_lib/variants/$v.so timeout 200 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/abb/test_$v.log 2>&1; echo "$v test rc=$?"
done
for wl in c2 32768x8 c2; do
  for v in default "$@"; do
    if [ $v = default ]; then unset FSP_LIB; else export FSP_LIB=paper_2412_01523_b200/_lib/variants/$v.so; fi
    echo "== $wl $v"; WL=$wl NOFA=1 timeout 90 python scripts/perf_attn.py 2>&1 | grep "fsp bwd\|rror"
  done
done > gpurun_out/abb/perf2.log 2>&1
cat gpurun_out/abb/perf2.log
