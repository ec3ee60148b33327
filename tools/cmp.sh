#!/bin/bash
# Compare libraries on the bench (3 runs each, 32 views): bash tools/cmp.sh libA.so libB.so ...
for lib in "$@"; do
  for i in 1 2 3; do
    FASTATLAS_LIB=$lib timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --profile-frames 0 \
      2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$lib'.split('/')[-1], 'value %.1f e2e %.1f latency %.4f' % (d['value'], d['e2e']['value'], d['ms_per_frame']))"
  done
done
