# A/B of tree-kernel variants (KOP_LIB) on the multi-EE beam and the generic tree solve, plus tree parity.
mkdir -p gpurun_out
for v in "" build/ab/tb1.so build/ab/tb2.so; do
  for p in fp32 fp64; do
    echo "lib=${v:-intree} $p beam: $(KOP_LIB=$v PREC=$p NHUM=100000 REPS=3 python tools/tree_beam_time.py 2>&1 | tail -1)"
  done
  echo "lib=${v:-intree} solve: $(KOP_LIB=$v python tools/tree_time.py 2>&1 | tail -2 | tr '\n' ' ')"
done
KOP_LIB=build/ab/tb2.so python -m pytest tests/test_gpu_tree.py -q -x 2>&1 | tail -3
