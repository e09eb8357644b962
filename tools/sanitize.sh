# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck, synccheck
# (logs: gpurun_out/r2_san_<tool>.log; copied to profiles/ when clean)
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py \
  > gpurun_out/r2_san_memcheck.log 2>&1; echo memcheck rc=$?
timeout 1800 $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_cases.py --no-k12 \
  > gpurun_out/r2_san_racecheck.log 2>&1; echo racecheck rc=$?
timeout 1200 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py --no-k12 \
  > gpurun_out/r2_san_synccheck.log 2>&1; echo synccheck rc=$?
