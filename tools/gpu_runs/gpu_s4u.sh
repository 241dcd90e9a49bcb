#!/bin/bash
# C2 lanes x reserved SMs on the final code
mkdir -p gpurun_out
for L in 3 4 5 6; do for r in 36 44 52; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --lanes $L --reserve-sms $r > gpurun_out/s4u_c2_${L}_$r.json 2>/dev/null
grep "^{" gpurun_out/s4u_c2_${L}_$r.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes $L reserve $r', round(d['value']), round(d['e2e']['value']), round(d['roofline']['scan_ms_avg'],3), d['clocks']['sm_mhz'])"
done; done
