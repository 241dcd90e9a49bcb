for rep in 1 2 3; do for l in 4 6; do timeout 600 python bench.py --no-cpu-baseline --lanes $l > gpurun_out/sw_l${l}_$rep.json 2>/dev/null; done; done
