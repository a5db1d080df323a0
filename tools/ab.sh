#!/usr/bin/env bash
# A/B of library builds on the GPU box: one short bench line per (config,
# build) with per-kernel times. Builds: the in-tree library ("new"),
# build/libqgm_old.so (OLD=1) and build/var_<v>.so (VARS="v1 v2", made by
# tools/build_variant.sh) and the in-tree library under environment knobs
# (ENVS="tag:VAR=value ..."). Usage: CFGS="C3shard C2" VARS="d32" bash tools/ab.sh
set -u
cd /root/repo
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $CFG --steps 3 --warmup 2 --check off --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); k=d['kernels_ms_per_launch']
print('$tag', '$CFG', d['ms_per_step'], 'join', k.get('k_join'), 'val', k.get('k_validate'), 'P', k.get('k_part_hist'), k.get('k_part_scatter'), k.get('k_refine_scatter'), 'e2e', round(d['e2e']['ms_per_step'],3), 'sort', d['stages_ms_per_step'].get('sort_unique'), 'strata', k.get('k_strata_seg'), d['counts']['hits'])"; }
for CFG in ${CFGS:-C3shard C2 C1}; do
run new X=1
[ -n "${OLD:-}" ] && run old QGM_LIB=/root/repo/build/libqgm_old.so
for v in ${VARS:-}; do run $v QGM_LIB=/root/repo/build/var_$v.so; done
for e in ${ENVS:-}; do run ${e%%:*} ${e#*:}; done
done
