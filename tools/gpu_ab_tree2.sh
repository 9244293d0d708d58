# A/B: in-tree library vs build/ab/tb4.so (A over the J mirror, 5 CTAs/SM) on the tree kernels, plus tree parity on tb4.
mkdir -p gpurun_out
for v in "" build/ab/tb4.so "" build/ab/tb4.so; do
  for p in fp32 fp64; do
    echo "lib=${v:-intree} $p beam: $(KOP_LIB=$v PREC=$p NHUM=100000 REPS=3 python tools/tree_beam_time.py 2>&1 | tail -1)"
  done
  echo "lib=${v:-intree} solve32: $(KOP_LIB=$v PREC=fp32 python tools/tree_time.py 2>&1 | head -1)"
  echo "lib=${v:-intree} solve64: $(KOP_LIB=$v PREC=fp64 python tools/tree_time.py 2>&1 | head -1)"
done
KOP_LIB=build/ab/tb4.so python -m pytest tests/test_gpu_tree.py tests/test_gpu_random_robots.py -q -x 2>&1 | tail -3
