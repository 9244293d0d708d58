# A/B: trajectory solve with two J-evaluation sites (in-tree) vs one (build/ab/ts2.so), interleaved, 10K trajectories.
mkdir -p gpurun_out
NTRAJ=10000 PREC=fp32 REPS=2 python tools/traj_time.py > /dev/null 2>&1
for v in "" build/ab/ts2.so "" build/ab/ts2.so; do
  for p in fp32 fp64; do
    echo "lib=${v:-intree} $p: $(KOP_LIB=$v NTRAJ=10000 PREC=$p REPS=3 python tools/traj_time.py 2>&1 | tail -1)"
  done
done
KOP_LIB=build/ab/ts2.so python -m pytest tests/test_gpu_traj.py -q -x 2>&1 | tail -2
