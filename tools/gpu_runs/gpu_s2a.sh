#!/bin/bash
# session-2 re-entry check: full GPU suite, C2/C4/C5 bench lines at HEAD
mkdir -p gpurun_out
export GIFT_PARITY_OUT=gpurun_out/s2a_parity.jsonl
rm -f $GIFT_PARITY_OUT
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/s2a_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/s2a_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2a_c2.json 2> gpurun_out/s2a_c2.err; echo c2=$?
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/s2a_c5.json 2> gpurun_out/s2a_c5.err; echo c5=$?
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2a_c4.json 2> gpurun_out/s2a_c4.err; echo c4=$?
for f in c2 c5 c4; do tail -1 gpurun_out/s2a_$f.json | head -c 600; echo; done
