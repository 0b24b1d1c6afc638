#!/bin/bash
for mb in ${CHUNKS:-20 40 80 120 200}; do
  echo -n "chunk ${mb}MB: "
  GK_CHUNK_MB=$mb python tools/quick_timing.py sh03b 3 | python -c "import json,sys; d=json.load(sys.stdin); print(d['nonlinear'])"
done
