# A/B of the forward pair kernel: default build vs the FSP_FWD_WG3=1 variant
# (scripts/build_variant.sh wg3 -DFSP_FWD_WG3=1), parity then timings.
mkdir -p gpurun_out/ab
V=paper_2412_01523_b200/_lib/variants/wg3.so
FSP_LIB=$V timeout 150 python -m pytest tests/test_gpu_attention.py -x -q -k "fwd" > gpurun_out/ab/test_wg3.log 2>&1; echo test rc=$?
tail -3 gpurun_out/ab/test_wg3.log
if grep -q passed gpurun_out/ab/test_wg3.log && ! grep -q failed gpurun_out/ab/test_wg3.log; then
for wl in c2 1024x256 4096x64 32768x8 c2; do
  for lib in default $V; do
    if [ $lib = default ]; then unset FSP_LIB; else export FSP_LIB=$lib; fi
    echo "== $wl $lib"; WL=$wl NOFA=1 timeout 90 python scripts/perf_attn.py 2>&1 | grep "fwd\|rror"
  done
done > gpurun_out/ab/perf.log 2>&1
cat gpurun_out/ab/perf.log
fi
