#!/bin/bash
# new S-IF bucket default: S-IF / C5 tests, C5 bench, then ncu of C5's S-IF kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -k "c5 or sif or rerank or top_k" > gpurun_out/s4m_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/s4m_tests.log
timeout 900 python bench.py --config c5 > gpurun_out/s4m_c5.json 2> gpurun_out/s4m_c5.err; echo c5=$?
grep "^{" gpurun_out/s4m_c5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value']), round(d['e2e']['value']), d['roofline'])"
bash tools/gpu_runs/gpu_s4l.sh
