set -x
for ck in 4 16; do
for dbg in 3 11 15; do
GIFT_TC_CHUNK_KB=$ck GIFT_TC_DBG=$dbg timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner > gpurun_out/st_c4s_ck${ck}_${dbg}.json 2> /dev/null; echo st=$?
done; done
