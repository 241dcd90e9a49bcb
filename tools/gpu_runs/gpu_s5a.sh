#!/bin/bash
# session 5: HEAD check on a rebuilt tree (GPU suite + smoke + default bench) then the C4 lanes x reserved-SM sweep
mkdir -p gpurun_out
export GIFT_REFSUITE_OUT=gpurun_out/s5a_reference_suite.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/s5a_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s5a_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/s5a_tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5a_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/s5a_smoke.log
timeout 900 python bench.py > gpurun_out/s5a_c2.json 2> gpurun_out/s5a_c2.err; echo c2=$?
grep "^{" gpurun_out/s5a_c2.json | tail -1 | cut -c1-300
for a in "1 0" "2 12" "2 20" "2 28" "3 20"; do set -- $a
timeout 600 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/s5a_c4_$1_$2.json 2>/dev/null
grep "^{" gpurun_out/s5a_c4_$1_$2.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes $1 reserve $2', round(d['value']), round(d['e2e']['value']), round(d['roofline']['scan_ms_avg'],2), d['clocks']['sm_mhz'])"
done
