set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "compressed_tile" > gpurun_out/cts_test.log 2>&1; echo cts=$?
for dbg in 0 64; do
GIFT_CTS=1 GIFT_TC_DBG=$dbg timeout 300 python tools/stage_profile.py --config c2 --steps 5 --reduce range > gpurun_out/st_c2_cts_$dbg.json 2> /dev/null; echo st=$?
done
