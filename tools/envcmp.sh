#!/bin/bash
# Compare environment settings on the bench (3 runs each, 32 views):
#   bash tools/envcmp.sh "FASTATLAS_PDL=0" "FASTATLAS_PDL=1"
for setting in "$@"; do
  for i in $(seq 1 ${REPS:-3}); do
    env $setting timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --profile-frames 3 \
      2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
st=d.get('stage_ms') or {}
print('$setting', 'value %.1f e2e %.1f latency %.4f depth %.1f vis %.1f' % (d['value'], d['e2e']['value'], d['ms_per_frame'], 1000*st.get('depth pass',0), 1000*st.get('visibility pass',0)))"
  done
done
