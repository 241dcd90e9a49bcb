# C4 scan: drain 4 vs 8 (compensated), after the epilogue-group race fix
set -x
for kb in 4 8; do
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --drain-kb $kb > gpurun_out/r2h_c4_d$kb.json 2> gpurun_out/r2h_c4_d$kb.err; echo c4_$kb=$?
done
