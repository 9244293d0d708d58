# Round-end refresh on one B200: GPU tests, smoke, widened-config timings, flop counts, trajectory ncu.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
python tools/widened_flops.py run > gpurun_out/wf.log 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --csv --log-file gpurun_out/wf.csv python tools/widened_flops.py run > gpurun_out/wf_ncu.log 2>&1; echo "wf rc=$?"
NTRAJ=296 REPS=1 python tools/traj_time.py > gpurun_out/tt.log 2>&1 && \
NTRAJ=296 REPS=1 ncu --set full --clock-control none --import-source on -k regex:k_traj_solve -c 1 -f -o gpurun_out/traj python tools/traj_time.py > gpurun_out/traj_ncu.log 2>&1; echo "trajncu rc=$?"
