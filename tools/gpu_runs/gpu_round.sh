# one gpurun call: parity tests of the new bundle format, C4 (1M shapes) bench, ncu captures
set -x
timeout 600 python -m pytest tests/test_bundle_format.py -x -q > gpurun_out/pytest_bundle.log 2>&1; echo pytest=$?
timeout 1800 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/bench_c4.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 40 -c 1 -o gpurun_out/scan_tc_c2 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_approx_tc -s 80 -c 1 -o gpurun_out/quant_tc_c2 $CMD > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
CMD4="python bench.py --config c4s --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD4 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4s.csv $CMD4 > gpurun_out/ncu4.log 2>&1; echo ncu4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 100 -c 1 -o gpurun_out/scan_tc_c4s $CMD4 > gpurun_out/ncu5.log 2>&1; echo ncu5=$?
