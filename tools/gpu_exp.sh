timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python tools/stage_profile.py --config c2 --steps 5 --kernels --reduce range --no-quantize > gpurun_out/stage_c2.log 2>&1; echo st=$?
timeout 300 python tools/quant_flags.py c2 > gpurun_out/qf.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?
