#!/bin/bash
# C1 graph lanes x reserved SMs
mkdir -p gpurun_out
for r in 44 0 20; do for L in 4 6 8 12; do
timeout 600 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --graph on --lanes $L --reserve-sms $r > gpurun_out/s4e_c1_${r}_$L.json 2> gpurun_out/s4e_c1_${r}_$L.err
tail -1 gpurun_out/s4e_c1_${r}_$L.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('reserve $r lanes $L', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4))" || tail -3 gpurun_out/s4e_c1_${r}_$L.err
done; done
