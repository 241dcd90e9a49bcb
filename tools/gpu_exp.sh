timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for dbg in 0 1; do GIFT_TC_DBG=$dbg timeout 900 python tools/stage_profile.py --config c4s --steps 3 --reduce owner > gpurun_out/c4s_sp_dbg$dbg.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1500 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
