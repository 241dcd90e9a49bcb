#!/bin/bash
# C3 e2e: whole query set (16 batches) vs the timed steps' batches (--steps 16 path), twice
mkdir -p gpurun_out
for a in "8 3" "16 3" "8 3"; do set -- $a
timeout 1800 python bench.py --config c3 --steps $1 --warmup $2 --no-cpu-baseline > gpurun_out/s4p_c3_$1.json 2> gpurun_out/s4p_c3_$1.err
grep "^{" gpurun_out/s4p_c3_$1.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 steps $1', round(d['value']), d['e2e'], d['clocks'])"
done
