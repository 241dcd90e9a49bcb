#!/bin/bash
# final HEAD: full GPU suite + smoke + default bench line
mkdir -p gpurun_out
export GIFT_REFSUITE_OUT=gpurun_out/s4w_reference_suite.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s4w_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s4w_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/s4w_tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4w_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/s4w_smoke.log
timeout 900 python bench.py > gpurun_out/s4w_c2.json 2> gpurun_out/s4w_c2.err; echo c2=$?
grep "^{" gpurun_out/s4w_c2.json | tail -1 | cut -c1-400
