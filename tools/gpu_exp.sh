set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python tools/stage_profile.py --config c4s --steps 3 --reduce owner --kernels > gpurun_out/st_c4s_ow.json 2> /dev/null; echo st=$?
timeout 1500 python tools/stage_profile.py --config c3 --steps 3 --reduce owner --kernels > gpurun_out/st_c3_ow.json 2> /dev/null; echo st=$?
