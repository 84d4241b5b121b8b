#!/bin/bash
# A/B of backward-kernel build knobs against the default build. Variants are built with
# scripts/build_variant.sh NAME -D...; run as: bash scripts/ab_bwd_knobs.sh OUTDIR NAME [NAME ...]
# (round 1: ring4, cw8, cw4, red8; round 2: poly4/poly2 -DFSP_BWD_POLY_EVERY=4/2,
# red8u -DFSP_BWD_REDUCE_WARPS=8 -DFSP_BWD_REDUCE_SPLIT=1). Parity, then C2 / 32K timings.
out=$1; shift
mkdir -p $out
for v in "$@"; do
  FSP_LIB=paper_2412_01523_b200/_lib/variants/$v.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q -k "bwd or one_token or flash" > $out/test_$v.log 2>&1; echo "$v test rc=$?"
done
for wl in c2 32768x8 c2 32768x8; do
  for v in default "$@"; do
    if [ $v = default ]; then unset FSP_LIB; else export FSP_LIB=paper_2412_01523_b200/_lib/variants/$v.so; fi
    echo "== $wl $v"; WL=$wl NOFA=1 timeout 90 python scripts/perf_attn.py 2>&1 | grep "fsp bwd\|rror"
  done
done > $out/perf.log 2>&1
cat $out/perf.log
