set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "evaluate_index or exact_ranking" > gpurun_out/pytest_eval.log 2>&1; echo pytest=$?
