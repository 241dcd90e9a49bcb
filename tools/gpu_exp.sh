GIFT_CTS=1 GIFT_TC_DBG=64 timeout 900 python bench.py --no-cpu-baseline --lanes 1 > gpurun_out/c2_cts64.json 2> gpurun_out/c2_cts64.err
GIFT_CTS=1 GIFT_TC_DBG=3 timeout 900 python bench.py --no-cpu-baseline --lanes 1 > gpurun_out/c2_cts3.json 2> gpurun_out/c2_cts3.err
GIFT_CTS=1 GIFT_TC_DBG=67 timeout 900 python bench.py --no-cpu-baseline --lanes 1 > gpurun_out/c2_cts67.json 2> gpurun_out/c2_cts67.err
