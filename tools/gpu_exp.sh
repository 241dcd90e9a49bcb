set -x
for pair in 0 1 0 1; do
GIFT_TC_PAIR=$pair timeout 600 python bench.py --steps 10 --no-cpu-baseline >> gpurun_out/bench_c2_pp.json 2> /dev/null; echo b2=$?
done
