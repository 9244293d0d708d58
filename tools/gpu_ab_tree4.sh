# A/B: FP64 multi-EE beam stage 1 with 4-warp CTAs (in-tree, 2 CTAs = 8 warps/SM) vs 9-warp CTAs (build/ab/w64_9.so, 1 CTA = 9 warps/SM), interleaved.
mkdir -p gpurun_out
PREC=fp32 REPS=3 python tools/tree_beam_time.py > /dev/null 2>&1
for v in "" build/ab/w64_9.so "" build/ab/w64_9.so; do
  echo "lib=${v:-intree} fp64 beam: $(KOP_LIB=$v PREC=fp64 NHUM=100000 REPS=5 python tools/tree_beam_time.py 2>&1 | tail -1)"
done
KOP_LIB=build/ab/w64_9.so python -m pytest tests/test_gpu_tree.py -q -x 2>&1 | tail -2
