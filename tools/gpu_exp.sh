set -x
C4="python tools/stage_profile.py --config c4s --steps 1 --reduce owner"
timeout 300 $C4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fif_scan_tc -s 99 -c 1 -o gpurun_out/scan_c4s_src $C4 > gpurun_out/ncu_src.log 2>&1; echo s4=$?
