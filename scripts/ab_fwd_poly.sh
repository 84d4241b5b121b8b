# With the three-warpgroup forward: full GPU suite on the default build, then the share of
# exponentials run on the FMA pipe (FSP_POLY_EVERY variants) A/B.
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/ab/pytest_gpu.log
for wl in c2 1024x256 32768x8; do
  for lib in default poly0 poly3 poly2; do
    if [ $lib = default ]; then unset FSP_LIB; else export FSP_LIB=paper_2412_01523_b200/_lib/variants/$lib.so; fi
    echo "== $wl $lib"; WL=$wl NOFA=1 timeout 90 python scripts/perf_attn.py 2>&1 | grep "fwd\|rror"
  done
done > gpurun_out/ab/poly.log 2>&1
cat gpurun_out/ab/poly.log
