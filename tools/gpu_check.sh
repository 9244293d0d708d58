#!/bin/bash
# Round-end refresh on one B200 (run under gpurun): GPU tests, smoke, the bench line (our arm and
# the reference arm).  Replaces round 1's gpu_final / gpu_refresh* scripts.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"
tail -n 2 gpurun_out/gpu_tests.log
