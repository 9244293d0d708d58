# After a tree-kernel change: GPU tests, widened-config lines, multi-EE beam ncu.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for p in fp32 fp64; do PREC=$p REPS=3 python tools/tree_beam_time.py; done > gpurun_out/tree_beam.log 2>&1
for p in fp32 fp64; do PREC=$p python tools/tree_time.py; done > gpurun_out/tree_time.log 2>&1
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
NHUM=4000 REPS=1 ncu --set full --clock-control none --import-source on -k regex:k_tree_beam_stage1 -c 1 -f -o gpurun_out/tree_beam python tools/tree_beam_time.py > gpurun_out/tb_ncu.log 2>&1; echo "tbncu rc=$?"
