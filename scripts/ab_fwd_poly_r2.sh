# forward exponent split A/B: FSP_POLY_EVERY = 4 (default) vs 2 / 3 / 6, C2 and 8 x 32K, two passes
V=paper_2412_01523_b200/_lib/variants
for v in fpoly2 fpoly3 fpoly6; do
  FSP_LIB=$V/$v.so timeout 200 python -m pytest tests/test_gpu_attention.py -x -q -k "fwd or one_token or flash or golden" > gpurun_out/r2al_test_$v.log 2>&1; echo "$v test rc=$?"
done
for wl in c2 32768x8 4096x64 c2 32768x8 4096x64; do
  for v in default fpoly2 fpoly3 fpoly6; do
    if [ $v = default ]; then unset FSP_LIB; else export FSP_LIB=$V/$v.so; fi
    echo "== $wl $v"; WL=$wl NOFA=1 CUDNN=0 timeout 60 python scripts/perf_attn.py 2>&1 | grep "fsp fwd\|rror"
  done
done
