#!/bin/bash
# A/B the step's field stage (fused field moment + int8 B slices) across variant libraries:
#   tools/field_ab.sh "" "GK_LIB_PATH=build/variants/libgk_x.so"
for cfg in "$@"; do
  echo -n "[$cfg] "
  env $cfg python bench.py --no-cpu-baseline --no-e2e --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), {k: round(v*1e3,3) for k,v in d['split_s'].items()})"
done
