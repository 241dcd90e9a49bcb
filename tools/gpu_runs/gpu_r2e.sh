# full GPU suite (incl. config scale), new bench: c2 gift arm, reference arm, c5 (single + shard1)
set -x
export GIFT_PARITY_OUT=gpurun_out/r2e_parity.jsonl
rm -f $GIFT_PARITY_OUT
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2e_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_c2.json 2> gpurun_out/r2e_c2.err; echo c2=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2e_ref.json 2> gpurun_out/r2e_ref.err; echo ref=$?
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/r2e_c5.json 2> gpurun_out/r2e_c5.err; echo c5=$?
timeout 900 python bench.py --config c4s --shard --steps 5 --warmup 3 > gpurun_out/r2e_c4s_shard.json 2> gpurun_out/r2e_c4s_shard.err; echo c4s_shard=$?
