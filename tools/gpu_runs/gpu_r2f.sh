# exact-matching tests, drain/compensation error study, c4s shard smoke, C4 bench
set -x
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q -m gpu > gpurun_out/r2f_pytest.log 2>&1; echo pytest=$?
timeout 900 python tools/drain_error.py > gpurun_out/r2f_drain.log 2>&1; echo drain=$?
timeout 900 python bench.py --config c4s --shard --steps 5 --warmup 3 > gpurun_out/r2f_c4s_shard.json 2> gpurun_out/r2f_c4s_shard.err; echo shard=$?
