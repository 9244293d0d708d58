# GPU tests, trajectory timing, executed-flop recount, then the widened-config lines against the new counts.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for p in fp32 fp64; do PREC=$p python tools/traj_time.py; done > gpurun_out/traj_time.log 2>&1; echo "traj rc=$?"
python tools/widened_flops.py run > gpurun_out/wf.log 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --csv --log-file gpurun_out/wf.csv python tools/widened_flops.py run > gpurun_out/wf_ncu.log 2>&1 && \
python tools/widened_flops.py parse gpurun_out/wf.csv > gpurun_out/wf_parse.log 2>&1 && cp profiles/r01_widened_flops.json gpurun_out/; echo "wf rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
