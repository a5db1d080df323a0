#!/usr/bin/env bash
# One GPU call that refreshes the round's evidence for the current library:
# per-config ncu sums (copied into profiles/<round>/ so the bench lines pick up
# roofline.traffic), every config with parity, sanitizers, the K=20 C2 line
# and its ncu launch list. Usage (GPU box): bash tools/final_evidence.sh r02
set -u
cd "$(dirname "$0")/.."
round=${1:-r02}
mkdir -p gpurun_out
bash tools/ncu_all.sh "$round" > gpurun_out/ncu_all.log 2>&1
cp gpurun_out/profiles_"$round"/ncu_*.json profiles/"$round"/ 2>/dev/null
bash tools/run_configs.sh > gpurun_out/run_configs.log 2>&1
bash tools/sanitize.sh memcheck racecheck synccheck > gpurun_out/sanitize.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_final.json 2> gpurun_out/bench_c2_final.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv \
  python bench.py --steps 2 --warmup 3 --check off --no-cpu > /dev/null 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c2_final.json 2>/dev/null
cat gpurun_out/ncu_all.log gpurun_out/run_configs.log gpurun_out/sanitize_summary.txt
