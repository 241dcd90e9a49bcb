# pair (cta_group::2) scan for fp16-exact queries: correctness + C4 speed; sharded world-1 shortcut
set -x
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q -m gpu -k "fp16 or variants or tensor_core" > gpurun_out/r2m_pytest.log 2>&1; echo pytest=$?
timeout 1500 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --pair on > gpurun_out/r2m_c4_pair.json 2> gpurun_out/r2m_c4_pair.err; echo c4pair=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29612 bench.py --config c4s --gpus 1 --shard --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_c4s_trs.json 2> gpurun_out/r2m_c4s_trs.err; echo trs=$?
timeout 900 python bench.py --config c5 --shard --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_c5s.json 2> gpurun_out/r2m_c5s.err; echo c5s=$?
