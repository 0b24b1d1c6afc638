#!/bin/bash
# time the sh03b nonlinear term under each ycol variant (VARS="0 5 6")
for v in ${VARS:-0 1 2 3 4 5 6}; do
  echo -n "variant $v: "
  GK_YCOL_VARIANT=$v python tools/quick_timing.py sh03b 3 | python -c "import json,sys; d=json.load(sys.stdin); print(d['nonlinear'])"
done
