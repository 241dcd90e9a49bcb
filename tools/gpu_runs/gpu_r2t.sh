# C2 lanes / reserved-SM sweep with the round-2 code (two runs each)
set -x
for cfg in "4 44" "4 36" "4 52" "3 44" "5 44" "4 28"; do set -- $cfg
for r in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/r2t_c2_l$1_r$2_$r.json 2> /dev/null; echo l$1_r$2_$r=$?
done; done
