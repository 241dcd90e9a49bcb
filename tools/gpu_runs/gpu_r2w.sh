set -x
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2w_memcheck.log 2>&1; echo memcheck=$?
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2w_racecheck.log 2>&1; echo racecheck=$?
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2w_synccheck.log 2>&1; echo synccheck=$?
