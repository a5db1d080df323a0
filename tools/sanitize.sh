#!/usr/bin/env bash
# compute-sanitizer over the device path: memcheck,
# racecheck (shared-memory hazards of the mbarrier/TMA join pipeline, the
# partition's staged counting sorts, the validation parking), synccheck and
# initcheck, each on tools/sanitize_workload.py (small inputs that still reach
# every kernel variant: warp-specialised and plain join, u16 counter hand-off,
# parked two-phase validation, strata radix path, CIGAR, streamed batches).
# Logs: gpurun_out/sanitize_<tool>.log.  Usage (GPU box):
#   bash tools/sanitize.sh [tool ...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tools=("$@")
[ ${#tools[@]} -eq 0 ] && tools=(memcheck racecheck synccheck initcheck)
for t in "${tools[@]}"; do
  extra=()
  [ "$t" = memcheck ] && extra=(--leak-check no)
  [ "$t" = racecheck ] && extra=(--racecheck-report hazard --num-cuda-barriers 16)
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool "$t" "${extra[@]}" --error-exitcode 9 --print-limit 200 \
    python tools/sanitize_workload.py > "gpurun_out/sanitize_$t.log" 2>&1
  echo "$t exit=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 "gpurun_out/sanitize_$t.log" | tee -a gpurun_out/sanitize_summary.txt
done
