set -x
C2="python tools/stage_profile.py --config c2 --steps 1 --reduce range"
C4="python tools/stage_profile.py --config c4s --steps 1 --reduce owner"
timeout 300 $C2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 40 -c 1 -o gpurun_out/q_scan_c2 $C2 > gpurun_out/ncu_a.log 2>&1; echo a=$?
timeout 900 ncu --set full --clock-control none -k regex:quant_approx_tc -s 80 -c 1 -o gpurun_out/q_quant_c2 $C2 > gpurun_out/ncu_b.log 2>&1; echo b=$?
timeout 300 $C4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 196 -c 1 -o gpurun_out/q_scan_c4s $C4 > gpurun_out/ncu_c.log 2>&1; echo c=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:quant_approx_tc --csv --log-file gpurun_out/quant_list.csv $C2 > gpurun_out/ncu_d.log 2>&1; echo d=$?
