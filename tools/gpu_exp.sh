set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner,gather,range --kernels > gpurun_out/stages_c4s.json 2> gpurun_out/stages_c4s.err; echo st4s=$?
timeout 300 python tools/stage_profile.py --config c2 --steps 3 --reduce owner,gather,range > gpurun_out/stages_c2.json 2> gpurun_out/stages_c2.err; echo st2=$?
timeout 900 python tools/stage_profile.py --config c4 --steps 3 --reduce owner,gather --kernels > gpurun_out/stages_c4.json 2> gpurun_out/stages_c4.err; echo st4=$?
