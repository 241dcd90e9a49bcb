set -x
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu > gpurun_out/r2v_edges.log 2>&1; echo edges=$?
