# round-2 full measurement set (current code): full GPU suite, every config's bench line, reference arm
set -x
export GIFT_PARITY_OUT=gpurun_out/fa_parity.jsonl
export GIFT_REFSUITE_OUT=gpurun_out/fa_refsuite.log
rm -f $GIFT_PARITY_OUT
timeout 3600 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/fa_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/fa_c2.json 2> gpurun_out/fa_c2.err; echo c2=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/fa_c1.json 2> gpurun_out/fa_c1.err; echo c1=$?
timeout 1500 python bench.py --config c3 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/fa_c3.json 2> gpurun_out/fa_c3.err; echo c3=$?
timeout 1800 python bench.py --config c4 --steps 8 --warmup 3 > gpurun_out/fa_c4.json 2> gpurun_out/fa_c4.err; echo c4=$?
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/fa_c5.json 2> gpurun_out/fa_c5.err; echo c5=$?
timeout 1500 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/fa_ref.json 2> gpurun_out/fa_ref.err; echo ref=$?
timeout 900 python bench.py --impl reference --config c1 --steps 5 --warmup 1 > gpurun_out/fa_ref_c1.json 2> gpurun_out/fa_ref_c1.err; echo refc1=$?
