for st in ${STAGES:-3 4 3 4}; do
  ADG_SCREEN_STAGES=$st timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('stages $st', d['value'], d['stages']['screen_kernel_ms'], d['clocks']['sm_mhz'])"
done
