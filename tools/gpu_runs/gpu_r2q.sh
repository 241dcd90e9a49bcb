set -x
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/r2q_pytest.log 2>&1; echo pytest=$?
timeout 1500 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2q_c4.json 2> gpurun_out/r2q_c4.err; echo c4=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2q_c2.json 2> gpurun_out/r2q_c2.err; echo c2=$?
timeout 900 python tools/scan_experiment.py c4s > gpurun_out/r2q_exp_c4s.log 2>&1; echo exp=$?
