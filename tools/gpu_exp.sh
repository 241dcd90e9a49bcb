set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce gather > gpurun_out/stages_c4s.json 2> gpurun_out/stages_c4s.err; echo st4s=$?
timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
timeout 300 python bench.py --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?
