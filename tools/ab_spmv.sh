#!/bin/bash
# A/B the headline SpMV across library variants (variants/<name>/libpencil_b200.so) on one box.
# usage: bash tools/ab_spmv.sh name1 name2 ...   ("base" = the in-tree library)
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib=variants/$v/libpencil_b200.so; fi
    PENCIL_B200_LIB=$lib timeout 200 python bench.py --no-suite --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), d['clocks']['reasons'])"
  done
done
