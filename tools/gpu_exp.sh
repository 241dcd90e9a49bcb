set -x
timeout 600 python bench.py --config c5 --steps 5 >> gpurun_out/b5_a.json 2> gpurun_out/b5_a.err; echo a=$?
timeout 600 python bench.py --config c5 --steps 5 >> gpurun_out/b5_a.json 2> /dev/null; echo a=$?
timeout 600 python bench.py --steps 10 >> gpurun_out/b2_a.json 2> gpurun_out/b2_a.err; echo c2=$?
timeout 900 python bench.py --config c4s --shard --steps 5 >> gpurun_out/b4s.json 2> gpurun_out/b4s.err; echo c4s=$?
