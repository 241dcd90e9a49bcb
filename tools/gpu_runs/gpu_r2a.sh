# round-2 check: GPU tests after the flag cleanup + fp16-exact scan shortcut, C2/C4 bench
set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_c2.json 2> gpurun_out/r2a_c2.err; echo c2=$?
timeout 1500 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_c4.json 2> gpurun_out/r2a_c4.err; echo c4=$?
