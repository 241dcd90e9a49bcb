# C4 with batches in flight (no host sync in the query path any more)
set -x
for cfg in "1 0" "2 20" "2 36" "3 36"; do set -- $cfg
timeout 1500 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --lanes $1 --reserve-sms $2 > gpurun_out/r2n_c4_l$1_r$2.json 2> gpurun_out/r2n_c4_l$1_r$2.err; echo c4_$1_$2=$?
done
