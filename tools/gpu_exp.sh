for sc in static dyn; do GIFT_TC_SCHED=$sc timeout 1500 python bench.py --config c3 --steps 8 --lanes 1 --no-cpu-baseline > gpurun_out/c3_$sc.json 2> gpurun_out/c3_$sc.err; done
