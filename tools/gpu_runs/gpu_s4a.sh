#!/bin/bash
# Session-4 measurement set on HEAD: GPU suite, smoke, every config's bench
# line, the reference arm, the C2 launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/s4a_gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/s4a_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s4a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/s4a_smoke.log
timeout 900 python bench.py > gpurun_out/s4a_c2.json 2> gpurun_out/s4a_c2.err; echo c2=$?
for c in c1 c5 c4 c3; do
timeout 1800 python bench.py --config $c > gpurun_out/s4a_$c.json 2> gpurun_out/s4a_$c.err; echo $c=$?
done
for c in c2 c1 c5 c4 c3; do
tail -1 gpurun_out/s4a_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d.get('roofline',{}).get('frac'), d['clocks'])"
done
timeout 1200 python bench.py --impl reference > gpurun_out/s4a_ref.json 2> gpurun_out/s4a_ref.err; echo ref=$?
tail -1 gpurun_out/s4a_ref.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4a_launches_c2.csv $CMD > gpurun_out/s4a_ncu.log 2>&1; echo ncu=$?
