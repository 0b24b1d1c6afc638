#!/bin/bash
# e2e A/B across env settings / libraries (same box, alternating):
#   tools/e2e_ab2.sh "GK_LIB_PATH=build/variants/libgk_old.so" "GK_E2E_VBLOCKS=4"
for cfg in "$@"; do
  echo -n "[$cfg] "
  env $cfg python bench.py --no-cpu-baseline --steps 3 --e2e-steps 6 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), round(d['e2e']['value']*1e3,2))"
done
