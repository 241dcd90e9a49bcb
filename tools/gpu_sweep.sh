for rep in 1 2 3; do for r in 52 64; do timeout 600 python bench.py --no-cpu-baseline --reserve-sms $r > gpurun_out/sw_r${r}_$rep.json 2>/dev/null; done; done
