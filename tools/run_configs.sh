#!/usr/bin/env bash
# Every BASELINE config through bench.py on one GPU with the parity check
# (GPU hit set vs the CPU path on the same reads, in a subprocess).
# Output: gpurun_out/cfg_<name>.json (one JSON line each) + .err.
#   bash tools/run_configs.sh [config[:check] ...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfgs=("$@")
[ ${#cfgs[@]} -eq 0 ] && cfgs=(C1:full C2:full C2best:full C2q12:sample C3:full C3shard:sample C4:full C4b64:full C5:sample C5m:full)
for spec in "${cfgs[@]}"; do
  name=${spec%%:*}
  check=${spec#*:}
  [ "$check" = "$spec" ] && check=sample
  steps=5; warm=3
  case $name in C3) steps=3; warm=1;; C5) steps=3; warm=1;; esac
  timeout ${CFG_TIMEOUT:-1500} python bench.py --config "$name" --steps $steps --warmup $warm --check "$check" \
    > "gpurun_out/cfg_$name.json" 2> "gpurun_out/cfg_$name.err"
  rc=$?
  python - "$name" "$rc" <<'EOF'
import json, sys
name, rc = sys.argv[1], sys.argv[2]
try:
    d = json.loads([l for l in open(f"gpurun_out/cfg_{name}.json") if l.startswith("{")][-1])
    p = d.get("parity") or {}
    print(f"{name} rc={rc} value={d['value']:.4g} ms/step={d['ms_per_step']} e2e={d['e2e']['value']:.4g} "
          f"parity={p.get('ok')} reads={p.get('reads')} gpu_hits={p.get('gpu_hits')} cpu_hits={p.get('cpu_hits')} "
          f"cpu={(d.get('cpu_baseline') or {}).get('value')}", flush=True)
except Exception as e:
    print(f"{name} rc={rc} no line ({e})", flush=True)
EOF
done
