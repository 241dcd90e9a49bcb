set -x
timeout 1800 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 600 python bench.py --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?
timeout 1800 python bench.py --config c3 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
