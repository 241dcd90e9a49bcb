set -x
GIFT_TC_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tensor_core_scan or fp16_storage or query_fif_vs_oracle or end_to_end" > gpurun_out/pair_acc.log 2>&1; echo pairacc=$?
nvidia-smi --query-gpu=name,memory.used --format=csv >> gpurun_out/pair_acc.log
GIFT_TC_PAIR=1 timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner > gpurun_out/stages_c4s_pair.json 2> gpurun_out/stages_c4s_pair.err; echo st4s=$?
GIFT_TC_PAIR=1 timeout 300 python tools/stage_profile.py --config c2 --steps 3 --reduce range > gpurun_out/stages_c2_pair.json 2> gpurun_out/stages_c2_pair.err; echo st2=$?
