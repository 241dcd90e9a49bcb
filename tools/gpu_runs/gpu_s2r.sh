#!/bin/bash
# calibrated truncation compensation: drain-interval error study (dense c4s + c2s), C4 bench at drain 4 / 8
mkdir -p gpurun_out
timeout 1500 python tools/drain_error.py > gpurun_out/s2r_drain_error.log 2>&1; echo drain=$?
python - <<'PY'
import json
for l in open('gpurun_out/drain_error.jsonl'):
    d=json.loads(l); print(d['case'], d['drain_kb'], d['compensated'], d['n'], '%.2e %.2e %.2e %.2e' % (d['max'], d['p9999'], d['mean_signed'], d['std_signed']))
PY
for kb in 4 8; do
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --drain-kb $kb > gpurun_out/s2r_c4_$kb.json 2> gpurun_out/s2r_c4_$kb.err; echo c4=$?
tail -1 gpurun_out/s2r_c4_$kb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 drain $kb', d['value'], d['e2e']['value'], r['scan_ms_avg'], r['frac'])"
done
