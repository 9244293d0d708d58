# Max-shared carveout preference on the big-smem kernels: repeated timings (the slow mode was intermittent).
mkdir -p gpurun_out
for i in 1 2 3; do
  PREC=fp32 REPS=4 python tools/tree_beam_time.py
  PREC=fp64 REPS=3 python tools/tree_beam_time.py
  PREC=fp32 python tools/traj_time.py
done > gpurun_out/carve.log 2>&1; echo "carve rc=$?"
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
