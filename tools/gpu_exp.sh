set -x
timeout 600 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
GIFT_TC_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tensor_core_scan or fp16_storage or end_to_end" > gpurun_out/el_acc_pair.log 2>&1; echo accp=$?
for dbg in 0 11; do
GIFT_TC_DBG=$dbg timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner > gpurun_out/st_c4s_e2_${dbg}.json 2> /dev/null; echo st=$?
done
timeout 300 python tools/stage_profile.py --config c2 --steps 3 --reduce range > gpurun_out/st_c2_e2.json 2> /dev/null; echo st=$?
