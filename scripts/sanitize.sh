#!/bin/bash
# compute-sanitizer over every FlexSP kernel (scripts/sanitize_run.py), one log per tool:
#   scripts/sanitize.sh OUTDIR [tool ...]     (default tools: memcheck racecheck synccheck initcheck)
# Only the library's kernels (mangled names in namespace fsp) are instrumented.
out=${1:-gpurun_out/sanitizer}; shift
tools=${@:-memcheck racecheck synccheck initcheck}
mkdir -p "$out"
cs=/usr/local/cuda/bin/compute-sanitizer
for tool in $tools; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  for c in pack a2a barrier fwd128 fwd128p fwd64 fwd64p fused; do
    echo "=== $tool $c" >> "$out/$tool.log"
    timeout 1200 $cs --tool $tool $extra --kernel-name regex=fsp --print-limit 20 \
      python scripts/sanitize_run.py $c >> "$out/$tool.log" 2>&1
    echo "rc=$?" >> "$out/$tool.log"
  done
done
