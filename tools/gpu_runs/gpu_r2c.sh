# qz4 (four D1 chunk buffers for fp16-exact queries): tests + C4 bench
set -x
timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q -m gpu -k "fp16 or tensor_core or variants" > gpurun_out/r2c_pytest.log 2>&1; echo pytest=$?
timeout 1500 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_c4.json 2> gpurun_out/r2c_c4.err; echo c4=$?
