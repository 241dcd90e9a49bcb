timeout 900 python -m pytest tests -m gpu -q -k "query_many" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?
