#!/bin/bash
# Both SpMV modes (tools/spmv_modes.py) across library variants, two rounds on one box.
# usage: bash tools/ab_spmv_modes.sh name1 name2 ...   ("base" = the in-tree library)
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib=variants/$v/libpencil_b200.so; fi
    echo "$v $(PENCIL_B200_LIB=$lib timeout 200 python tools/spmv_modes.py 2>/dev/null | tail -1)"
  done
done
