V=paper_2412_01523_b200/_lib/variants
for wl in 1024x256 4096x64 32768x8; do
  echo "== fwd timing $wl"; FSP_LIB=$V/fwdtime.so WL=$wl NOFA=1 CUDNN=0 timeout 90 python scripts/perf_attn.py 2>&1 | grep -v "^$" | head -4
  echo "== bwd timing $wl"; FSP_LIB=$V/bwdtime.so WL=$wl NOFA=1 CUDNN=0 timeout 90 python scripts/perf_attn.py 2>&1 | grep "bwd" | head -4
done
