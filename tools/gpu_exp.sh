timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/ingest_bench.py --shapes 2000 > gpurun_out/ingest.json 2> gpurun_out/ingest.err; echo ing=$?
