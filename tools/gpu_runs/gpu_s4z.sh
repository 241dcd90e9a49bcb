#!/bin/bash
# C4 lanes x reserved SMs on the final code
mkdir -p gpurun_out
for a in "1 0" "2 12" "2 20" "2 28" "3 20"; do set -- $a
timeout 900 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/s4z_c4_$1_$2.json 2>/dev/null
grep "^{" gpurun_out/s4z_c4_$1_$2.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes $1 reserve $2', round(d['value']), round(d['e2e']['value']), round(d['roofline']['scan_ms_avg'],2), d['clocks']['sm_mhz'])"
done
