#!/bin/bash
# compute-sanitizer over a small, complete pass of the kernels (tools/sanitize_probe.py), on the GPU box:
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
# (On the round-2 pool compute-sanitizer is closed — its wrapper refuses to run — so these option sets are covered
# there by running tools/sanitize_probe.py plainly and by the bit-exact GPU tests; the script is kept for boxes that allow it.)
# memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory hazards: the warp queues, the flushed
# 16-bit histogram, the record staging buffers, the direct form's staging buffers and Q3 / Q4 area, the per-CTA emit context) and synccheck (barriers inside the
# flush loop), each on the option sets that switch those paths on.  Output: gpurun_out/sanitize_*.log; exit code != 0
# when a tool reports anything.
set -u
out=gpurun_out
mkdir -p $out
rc=0
run() {  # tool fixture options
  local log=$out/sanitize_$1_$2_${3//[=,]/_}.log
  compute-sanitizer --tool $1 --error-exitcode 9 --print-limit 20 python tools/sanitize_probe.py $2 "$3" > $log 2>&1
  local r=$?
  echo "$1 $2 [$3]: rc=$r $(grep -c -E 'ERROR SUMMARY: 0 errors|RACECHECK SUMMARY: 0 hazards' $log) clean summaries; $(grep -E 'sanitize probe ok|SUMMARY' $log | tr '\n' ' ')"
  [ $r -ne 0 ] && rc=1
}
run memcheck cfg3_tess16_exact_trained ""
run memcheck cfg5_stars_scaled "stage_lut=1,hist16=1,strip_index=1"
run memcheck cfg4_tess36_approx1m_k56 "hist16=1,ids_late=1,tier_sub=1"
run memcheck cfg4_tess36_approx1m_k56 "hist16=1,direct=1,link_sub=1"
run racecheck cfg4_tess36_approx1m_k56 "hist16=1,direct=1,link_sub=1"
run racecheck cfg3_tess16_exact_trained ""
run racecheck cfg5_stars_scaled "stage_lut=1,hist16=1,strip_index=1"
run synccheck cfg5_stars_scaled "stage_lut=1,hist16=1"
exit $rc
