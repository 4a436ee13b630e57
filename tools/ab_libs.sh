#!/bin/bash
# A/B the default bench over tuning-variant libraries built by
#   python paper_2312_15554_b200/_build.py --variant NAME -DMACRO=VALUE ...
# usage: tools/ab_libs.sh "<bench args>" lib_a.so lib_b.so ...   ("default" = product library)
args="$1"; shift
for lib in "$@"; do
  if [ "$lib" = default ]; then unset POREFLOW_B200_LIB; else export POREFLOW_B200_LIB=$lib; fi
  python bench.py $args --no-cpu-baseline 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
s = d.get('stages', {})
print('$(basename $lib)', round(d['value'] / 1e9, 3), round(d['ms_per_step'], 4), {k: round(v['ms'], 3) for k, v in s.items()})"
done
