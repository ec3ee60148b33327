#!/bin/bash
# Pipelined throughput vs FramePipeline slots: bash tools/depthcmp.sh 4 6 8
for d in "$@"; do
  for i in $(seq 1 ${REPS:-2}); do
    timeout 300 python bench.py --no-cpu-baseline --profile-frames 0 --depth $d 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('depth $d', 'value %.1f e2e %.1f latency %.4f' % (d['value'], d['e2e']['value'], d['ms_per_frame']))"
  done
done
