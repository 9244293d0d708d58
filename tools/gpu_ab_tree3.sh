# A/B: in-tree library vs build/ab/tb6.so (one evaluation site per beam run: runtime J flag), interleaved, plus tree parity on tb6.
mkdir -p gpurun_out
PREC=fp32 REPS=3 python tools/tree_beam_time.py > /dev/null 2>&1  # clock warm-up
for v in "" build/ab/tb6.so "" build/ab/tb6.so; do
  for p in fp32 fp64; do
    echo "lib=${v:-intree} $p beam: $(KOP_LIB=$v PREC=$p NHUM=100000 REPS=3 python tools/tree_beam_time.py 2>&1 | tail -1)"
  done
done
KOP_LIB=build/ab/tb6.so python -m pytest tests/test_gpu_tree.py tests/test_gpu_random_robots.py -q -x 2>&1 | tail -3
