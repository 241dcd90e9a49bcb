timeout 900 python tools/kmeans_bench.py > gpurun_out/kmeans_bench.json 2> gpurun_out/kmeans_bench.err; echo km=$?
