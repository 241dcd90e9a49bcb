set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1800 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 600 python bench.py --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?
