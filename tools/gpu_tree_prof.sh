# Refresh the widened-config lines and capture the multi-EE IK-Beam stage-1 kernel under ncu.
mkdir -p gpurun_out
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
NHUM=4000 REPS=1 python tools/tree_beam_time.py > gpurun_out/tb_small.log 2>&1 && \
NHUM=4000 REPS=1 ncu --set full --clock-control none --import-source on -k regex:k_tree_beam_stage1 -c 1 -f -o gpurun_out/tree_beam python tools/tree_beam_time.py > gpurun_out/tb_ncu.log 2>&1; echo "tbncu rc=$?"
