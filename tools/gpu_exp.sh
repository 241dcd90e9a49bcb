set -x
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_streamed.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config c4s --shard --steps 5 > gpurun_out/bench_c4s_shard.json 2> gpurun_out/bench_c4s_shard.err; echo sh=$?
