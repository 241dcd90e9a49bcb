# GPU tests + ncu of the C4-shaped scan (c4s) after the fp16-exact shortcut
set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2b_pytest.log 2>&1; echo pytest=$?
CMD4="python bench.py --config c4s --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD4 > gpurun_out/r2b_c4s.json 2> gpurun_out/r2b_c4s.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 100 -c 1 -o gpurun_out/r2b_scan_c4s $CMD4 > gpurun_out/r2b_ncu.log 2>&1; echo ncu=$?
