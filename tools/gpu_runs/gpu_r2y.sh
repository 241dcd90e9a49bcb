CMD="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r2y_c5.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2y_launches_c5.csv $CMD > gpurun_out/r2y_ncu.log 2>&1; echo launches=$?
