set -x
GIFT_TC_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tensor_core_scan or fp16_storage or end_to_end or query_fif" > gpurun_out/pcb_acc.log 2>&1; echo acc=$?
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tensor_core_scan or fp16_storage or end_to_end" > gpurun_out/scb_acc.log 2>&1; echo acc=$?
for pair in 0 1; do
GIFT_TC_PAIR=$pair timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner > gpurun_out/st_c4s_pcb_${pair}.json 2> /dev/null; echo st=$?
GIFT_TC_PAIR=$pair GIFT_TC_DBG=11 timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner > gpurun_out/st_c4s_pcb11_${pair}.json 2> /dev/null; echo st=$?
done
