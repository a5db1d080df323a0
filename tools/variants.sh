#!/bin/bash
# Bench the current library and each build/variants/lib_<name>.so given as
# arguments (QGM_LIB override), printing ms/step and per-kernel times.
# Usage (on the GPU box): bash tools/variants.sh [name ...] [-- bench args]
names=(); extra=()
while [ $# -gt 0 ]; do if [ "$1" = "--" ]; then shift; extra=("$@"); break; fi; names+=("$1"); shift; done
for c in HEAD "${names[@]}"; do
  if [ "$c" = HEAD ]; then unset QGM_LIB; else export QGM_LIB=$PWD/build/variants/lib_$c.so; fi
  timeout 300 python bench.py --no-cpu "${extra[@]}" > gpurun_out/var_$c.json 2> gpurun_out/var_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/var_{c}.json"))
    print(c, d["ms_per_step"], d["e2e"]["ms_per_step"], d["counts"]["hits"], json.dumps(d["kernels_ms_per_launch"]))
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/var_{c}.err").read()[-800:])
PY
done
