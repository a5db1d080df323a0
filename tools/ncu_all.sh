#!/usr/bin/env bash
# ncu evidence for every bench config (GPU box): per-kernel DRAM bytes,
# instructions and durations of one map of the config's first batch, folded
# into profiles/<round>/ncu_<config>.json (bench.py reads them as roofline
# traffic when the library sha matches). Usage: bash tools/ncu_all.sh r02 [configs...]
set -u
cd "$(dirname "$0")/.."
round=$1; shift
cfgs=("$@")
[ ${#cfgs[@]} -eq 0 ] && cfgs=(C1 C2 C3shard C4 C4b64 C5m C2q12)
mkdir -p gpurun_out
for c in "${cfgs[@]}"; do
  timeout 900 ncu --profile-from-start off --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --csv --log-file gpurun_out/ncu_$c.csv python tools/ncu_capture.py run $c > /dev/null 2>&1
  python tools/ncu_capture.py parse $c gpurun_out/ncu_$c.csv gpurun_out/profiles_$round > /dev/null 2>&1 && echo "$c ok" || echo "$c failed"
done
