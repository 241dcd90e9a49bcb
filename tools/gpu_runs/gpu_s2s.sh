#!/bin/bash
# drain 8 default: full GPU suite, C2/C3/C4/C5 bench lines
mkdir -p gpurun_out
export GIFT_PARITY_OUT=gpurun_out/s2s_parity.jsonl
rm -f $GIFT_PARITY_OUT
timeout 2400 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/s2s_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/s2s_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2s_c2.json 2> gpurun_out/s2s_c2.err; echo c2=$?
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 > gpurun_out/s2s_c4.json 2> gpurun_out/s2s_c4.err; echo c4=$?
timeout 1500 python bench.py --config c3 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s2s_c3.json 2> gpurun_out/s2s_c3.err; echo c3=$?
for f in c2 c4 c3; do tail -1 gpurun_out/s2s_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"; done
