timeout 1500 python bench.py --config c3 --steps 8 --no-cpu-baseline --lanes 1 > gpurun_out/c3_l1.json 2>/dev/null
timeout 1500 python bench.py --config c3 --steps 8 --no-cpu-baseline --lanes 2 --reserve-sms 44 > gpurun_out/c3_l2r44.json 2>/dev/null
timeout 1500 python bench.py --config c3 --steps 8 --no-cpu-baseline --lanes 3 --reserve-sms 44 > gpurun_out/c3_l3r44.json 2>/dev/null
