#!/bin/bash
# quick GPU check: parity suite + bench stage summary
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms/frame %.4f  e2e %.1f atl/s' % (d['ms_per_frame'], d['e2e']['value']))
print({k: round(v*1000,1) for k,v in d['stage_ms'].items()})"
