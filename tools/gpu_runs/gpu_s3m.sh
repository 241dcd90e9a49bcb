#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k graphed > gpurun_out/s3m.log 2>&1; echo tests=$?
tail -3 gpurun_out/s3m.log
