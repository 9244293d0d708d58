#!/bin/bash
# The reference's own tests against the B200 package (staged by oracle/make_refsuite.py), on a B200.
mkdir -p gpurun_out
PYTHONPATH=oracle/_ref/refsuite:. python -m pytest oracle/_ref/refsuite/tests -q -rA -p no:cacheprovider \
    -o testpaths= --rootdir oracle/_ref/refsuite > gpurun_out/refsuite.log 2>&1
echo "refsuite rc=$?"
tail -n 3 gpurun_out/refsuite.log
