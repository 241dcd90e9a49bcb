set -x
timeout 900 python tools/scan_experiment.py c4s > gpurun_out/r2o_exp_c4s.log 2>&1; echo c4s=$?
timeout 900 python tools/scan_experiment.py c2 > gpurun_out/r2o_exp_c2.log 2>&1; echo c2=$?
