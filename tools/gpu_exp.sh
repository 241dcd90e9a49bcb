timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --config c5 --steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
