# host description of the GPU box + baseline GPU test run
set -x
lscpu > gpurun_out/lscpu.txt 2>&1
free -g > gpurun_out/free.txt 2>&1
nproc > gpurun_out/nproc.txt
python -c "import numpy; numpy.show_config()" > gpurun_out/np_config.txt 2>&1
python - > gpurun_out/blas_speed.txt 2>&1 <<'PY'
import numpy as np, time, os
a = np.random.rand(4096, 4096); b = np.random.rand(4096, 4096)
a @ b
t = time.time(); a @ b; dt = time.time() - t
print("dgemm 4096^3 GFLOP/s", 2 * 4096**3 / dt / 1e9, "cores", os.cpu_count())
PY
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_base.log 2>&1; echo pytest=$?
