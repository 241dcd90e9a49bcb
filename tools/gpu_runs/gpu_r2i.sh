# cheap per-item truncation compensation: error study, C4 + C2 bench, reference suite via the shim
set -x
timeout 900 python tools/drain_error.py > gpurun_out/r2i_drain.log 2>&1; echo drain=$?
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_c4.json 2> gpurun_out/r2i_c4.err; echo c4=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_c2.json 2> gpurun_out/r2i_c2.err; echo c2=$?
GIFT_REFSUITE_OUT=gpurun_out/r2i_refsuite.log timeout 1800 python -m pytest tests/test_gpu_reference_suite.py -x -q > gpurun_out/r2i_refsuite_pytest.log 2>&1; echo refsuite=$?
