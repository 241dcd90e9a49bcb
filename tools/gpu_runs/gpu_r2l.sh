# C3 bench (round-2 code); torchrun single-rank runs of the single-GPU and sharded paths; C5 sharded (world 1)
set -x
timeout 1500 python bench.py --config c3 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_c3.json 2> gpurun_out/r2l_c3.err; echo c3=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29611 bench.py --config c4s --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_c4s_tr.json 2> gpurun_out/r2l_c4s_tr.err; echo tr=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29612 bench.py --config c4s --gpus 1 --shard --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_c4s_trs.json 2> gpurun_out/r2l_c4s_trs.err; echo trs=$?
timeout 900 python bench.py --config c5 --shard --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_c5s.json 2> gpurun_out/r2l_c5s.err; echo c5s=$?
