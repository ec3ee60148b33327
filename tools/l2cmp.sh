for l2 in flush replicas; do for i in 1 2; do timeout 300 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --profile-frames 0 --l2 $l2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$l2', 'value %.1f e2e %.1f latency %.4f' % (d['value'], d['e2e']['value'], d['ms_per_frame']))"; done; done
