python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-shards 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phase_ms_serial'], d['roofline']['executed_achieved'])"
