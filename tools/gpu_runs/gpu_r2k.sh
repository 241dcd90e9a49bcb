# round-2 profiles: C2 bench command launch list + full capture of a timed scan; C4 drain 8 vs 4
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r2k_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches_c2.csv $CMD > gpurun_out/r2k_ncu1.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 45 -c 1 -o gpurun_out/r2k_scan_c2 $CMD > gpurun_out/r2k_ncu2.log 2>&1; echo full=$?
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --drain-kb 8 > gpurun_out/r2k_c4_d8.json 2> gpurun_out/r2k_c4_d8.err; echo c4d8=$?
CMD4="python bench.py --config c4s --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD4 > gpurun_out/r2k_plain4.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 100 -c 1 -o gpurun_out/r2k_scan_c4s $CMD4 > gpurun_out/r2k_ncu3.log 2>&1; echo full4=$?
