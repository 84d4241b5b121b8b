V=paper_2412_01523_b200/_lib/variants
for wl in 1024x256 c2 2048x128 1024x256 c2 2048x128; do
  for v in base default; do
    if [ $v = default ]; then unset FSP_LIB; else export FSP_LIB=$V/$v.so; fi
    for e in 0 1; do
      echo "== $wl $v early=$e"; FSP_FWD_EARLY=$e WL=$wl NOFA=1 CUDNN=0 timeout 90 python scripts/perf_attn.py 2>&1 | grep "fsp fwd\|rror"
    done
  done
done
for e in 0 1; do echo "== timing 1024x256 early=$e"; FSP_LIB=$V/fwdtime2.so FSP_FWD_EARLY=$e WL=1024x256 NOFA=1 CUDNN=0 timeout 90 python scripts/perf_attn.py 2>&1 | grep -v "^$" | head -8; done
