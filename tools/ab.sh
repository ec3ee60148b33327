#!/bin/bash
# A/B a runtime switch: bash tools/ab.sh VAR "v1 v2 ..." [kernel-regex]
# parity suite once, then per value: bench summary + warm launch-table lines
var=$1; vals=$2; pat=${3:-vis}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in $vals; do
  echo "== $var=$v"
  env $var=$v timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_size or camera_path" 2>&1 | tail -1
  env $var=$v timeout 600 python bench.py --steps 16 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('latency %.4f value %.1f e2e %.1f' % (d['ms_per_frame'], d['value'], d['e2e']['value']), {k: round(v*1000,1) for k,v in d['stage_ms'].items()})"
  env $var=$v bash tools/lt.sh ab_$v 2>&1 | grep -iE "$pat"
done
