#!/bin/bash
# Interleaved A/B timing of library builds on one B200 (run under gpurun).
#   LIBS="default variants/libkinoptik_b200_X.so" REPEAT=2 bash tools/gpu_ab.sh python tools/beam_time.py fp32
# "default" = the in-tree library.  Builds come from paper_2505_03728_b200._build.build(variant=NAME,
# defines=[...]) (-> variants/, shipped with the snapshot).  Runs are interleaved (A B A B ...) because
# the first timed calls on a fresh box can be slower; compare medians.
# Replaces round 1's one-off gpu_ab_* scripts.
mkdir -p gpurun_out
for i in $(seq ${REPEAT:-2}); do
  for L in ${LIBS:-default}; do
    if [ "$L" = default ]; then
      echo "lib=default $("$@" 2>&1 | tail -1)"
    else
      echo "lib=$L $(KOP_LIB=$L "$@" 2>&1 | tail -1)"
    fi
  done
done
