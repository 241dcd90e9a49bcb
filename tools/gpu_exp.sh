timeout 1500 python bench.py --config c3 --steps 8 --no-cpu-baseline > gpurun_out/c3_def.json 2> gpurun_out/c3_def.err
GIFT_SIF=rows timeout 1500 python bench.py --config c3 --steps 8 --no-cpu-baseline > gpurun_out/c3_rows.json 2> gpurun_out/c3_rows.err
