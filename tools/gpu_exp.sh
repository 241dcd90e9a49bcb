timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for dbg in 0 1; do GIFT_TC_DBG=$dbg timeout 900 python bench.py --config c4s --steps 5 --no-cpu-baseline > gpurun_out/c4s_dbg$dbg.json 2> gpurun_out/c4s_dbg$dbg.err; done
GIFT_TC_PAIR=0 timeout 600 python bench.py --no-cpu-baseline --lanes 1 > gpurun_out/bench_c2_single.json 2> gpurun_out/bench_c2_single.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
