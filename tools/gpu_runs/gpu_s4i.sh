#!/bin/bash
# graph regrowth test; C2 bench with the whole-query-set e2e; C5 split loads in flight (SB_U 4/8/12)
mkdir -p gpurun_out
#timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "graph" > gpurun_out/s4i_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s4i_tests.log
#timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s4i_c2.json 2> gpurun_out/s4i_c2.err; echo c2=$?
#tail -1 gpurun_out/s4i_c2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['value']), d['e2e'], d['clocks'])"
cp paper_1604_01879_b200/libgift.so /tmp/libgift_prod.so
for u in 4 8 12; do
if [ $u != 4 ]; then cp tools/libgift_sbu$u.so paper_1604_01879_b200/libgift.so; else cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so; fi
timeout 900 python bench.py --config c5 --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/s4i_c5_$u.json 2>gpurun_out/s4i_c5_$u.err; echo sbu$u=$?
grep "^{" gpurun_out/s4i_c5_$u.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SB_U $u', round(d['value']), round(d['e2e']['value']), d['roofline']['sif_ms_avg'])"
timeout 900 python bench.py --config c5 --steps 12 --warmup 3 --no-cpu-baseline --lanes 1 > gpurun_out/s4i_c5_${u}_l1.json 2>/dev/null
grep "^{" gpurun_out/s4i_c5_${u}_l1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SB_U $u lanes 1', round(d['value']), round(d['e2e']['value']), d['roofline']['sif_ms_avg'])"
done
cp /tmp/libgift_prod.so paper_1604_01879_b200/libgift.so
