set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/r2r_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config c4s --shard --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_c4s_shard.json 2> gpurun_out/r2r_c4s_shard.err; echo shard=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2r_c2.json 2> gpurun_out/r2r_c2.err; echo c2=$?
