#!/bin/bash
# C4 timeline: where one-lane steps spend time beyond the kernels' sum
mkdir -p gpurun_out
for L in 1 2; do
timeout 1500 python tools/lane_trace.py --config c4 --lanes $L --steps 8 > gpurun_out/s4b_trace_c4_l$L.json 2> gpurun_out/s4b_trace_c4_l$L.err; echo trace$L=$?
tail -1 gpurun_out/s4b_trace_c4_l$L.json
done
timeout 1500 python tools/stage_profile.py --config c4 > gpurun_out/s4b_stage_c4.json 2> gpurun_out/s4b_stage_c4.err; echo stage=$?
tail -1 gpurun_out/s4b_stage_c4.json
