# Round-end refresh: GPU tests, smoke, headline bench, widened-config lines, multi-EE beam launch list.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
NHUM=20000 REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tree_beam_launches.csv python tools/tree_beam_time.py > gpurun_out/tbl.log 2>&1; echo "tbl rc=$?"
