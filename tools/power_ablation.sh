for v in TCB_CARVE_DEBUG=0 TCB_CARVE_DEBUG=1 TCB_CARVE_DEBUG=2 TCB_CARVE_DEBUG=3 TCB_CARVE_MAXFREE=0; do
  env $v timeout 300 python bench.py --steps 300 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$v] layer', d['value'], 'carve', d['kernels_ms']['carve_fwd'], 'clk', d['clocks']['sm_mhz'], 'W', d['clocks']['power_w_median'])"
done
