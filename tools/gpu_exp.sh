timeout 900 python -m pytest tests -m gpu -q -x -k "query_many or sparse" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for l in 4; do timeout 600 python bench.py --lanes $l > gpurun_out/bench_c2_l$l.json 2> gpurun_out/bench_c2_l$l.err; done
for l in 1 2; do timeout 1200 python bench.py --config c4 --steps 5 --lanes $l --no-cpu-baseline > gpurun_out/bench_c4_l$l.json 2> gpurun_out/bench_c4_l$l.err; done
timeout 1200 python bench.py --config c3 --steps 8 --lanes 2 --no-cpu-baseline > gpurun_out/bench_c3_l2.json 2> gpurun_out/bench_c3_l2.err
timeout 1200 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
