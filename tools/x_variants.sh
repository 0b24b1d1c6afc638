#!/bin/bash
for v in 0 1 2 3; do
  echo -n "x-teams $v: "
  GK_X_TEAMS=$v python tools/quick_timing.py sh03b 3 | python -c "import json,sys; d=json.load(sys.stdin); print(d['nonlinear'])"
done
