timeout 900 python -m pytest tests/test_bundle_format.py tests/test_kmeans.py tests/test_ingest.py -q > gpurun_out/pytest_tb.log 2>&1; echo pytest=$?
