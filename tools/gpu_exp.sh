timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?
timeout 1200 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
timeout 900 python bench.py --config c4s --steps 5 --no-cpu-baseline > gpurun_out/bench_c4s.json 2> gpurun_out/bench_c4s.err; echo c4s=$?
