set -x
C2="python tools/stage_profile.py --config c2 --steps 1 --reduce range"
C4="python tools/stage_profile.py --config c4s --steps 1 --reduce owner"
timeout 300 $C2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stage_c2.csv $C2 > gpurun_out/ncu_l2.log 2>&1; echo l2=$?
timeout 300 $C4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stage_c4s.csv $C4 > gpurun_out/ncu_l4.log 2>&1; echo l4=$?
N2=$(grep -c fif_scan_tc gpurun_out/launches_stage_c2.csv); N4=$(grep -c fif_scan_tc gpurun_out/launches_stage_c4s.csv); echo n2=$N2 n4=$N4
S2=$((N2/2-3)); S4=$((N4/2-3))
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s $S2 -c 1 -o gpurun_out/r01_scan_c2 $C2 > gpurun_out/ncu_s2.log 2>&1; echo s2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s $S4 -c 1 -o gpurun_out/r01_scan_c4s $C4 > gpurun_out/ncu_s4.log 2>&1; echo s4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_approx_tc -s $S2 -c 1 -o gpurun_out/r01_quant_c2 $C2 > gpurun_out/ncu_q2.log 2>&1; echo q2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_owner_reduce -s $S4 -c 1 -o gpurun_out/r01_owner_c4s $C4 > gpurun_out/ncu_o4.log 2>&1; echo o4=$?
