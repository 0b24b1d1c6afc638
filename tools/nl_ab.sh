#!/bin/bash
# A/B the nonlinear kernel across env settings / variant libraries:
#   tools/nl_ab.sh "GK_Y144=cta" "" "GK_LIB_PATH=build/variants/libgk_x.so"
for cfg in "$@"; do
  echo -n "[$cfg] "
  env $cfg python tools/quick_timing.py sh03b 3 | python -c "import json,sys; d=json.load(sys.stdin); print(d['nonlinear'])"
done
