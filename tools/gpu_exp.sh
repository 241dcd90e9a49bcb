timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1500 python tools/lane_trace.py --config c4 --lanes 1 --steps 4 > gpurun_out/lt_c4_l1.json 2> gpurun_out/lt_c4_l1.err
timeout 1500 python tools/lane_trace.py --config c3 --lanes 1 --steps 4 > gpurun_out/lt_c3_l1.json 2> gpurun_out/lt_c3_l1.err
