# config-scale parity (C1 exact config, C2 64 queries x 10k + full oracle self-join, C5 50k x 1024q), sharded tests
set -x
export GIFT_PARITY_OUT=gpurun_out/r2d_parity.jsonl
rm -f $GIFT_PARITY_OUT
timeout 2400 python -m pytest tests/test_gpu_config_scale.py -x -q -s --durations=0 > gpurun_out/r2d_scale.log 2>&1; echo scale=$?
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_dist.py -x -q > gpurun_out/r2d_sharded.log 2>&1; echo sharded=$?
