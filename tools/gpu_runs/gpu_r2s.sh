set -x
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q -m gpu -k "fp16 or variants" > gpurun_out/r2s_pytest.log 2>&1; echo pytest=$?
timeout 1500 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2s_c4.json 2> gpurun_out/r2s_c4.err; echo c4=$?
timeout 900 python tools/scan_experiment.py c4s > gpurun_out/r2s_exp_c4s.log 2>&1; echo exp=$?
