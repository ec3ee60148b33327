#!/bin/bash
# quick GPU check: parity suite + bench stage summary
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 16 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('latency %.4f ms/frame  value %.1f atl/s (%.4f ms/step)  e2e %.1f atl/s' % (d['ms_per_frame'], d['value'], d['ms_per_step'], d['e2e']['value']))
print({k: round(v*1000,1) for k,v in d['stage_ms'].items()})"
