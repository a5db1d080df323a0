#!/usr/bin/env bash
# A/B of the API index build (qgm_index_build, C2 batch) across library
# builds: the in-tree library ("new"), build/var_<v>.so for VARS="v1 v2".
#   VARS="hd" bash tools/ib_ab.sh
cd /root/repo
for rep in 1 2; do
for v in new ${VARS:-}; do
  L=""; [ $v != new ] && L=/root/repo/build/var_$v.so
  QGM_LIB=$L timeout 300 python bench.py --config C2 --steps 3 --warmup 2 --check off --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', d['index_build']['ms'], d['index_build']['frac'], d['ms_per_step'])"
done
done
