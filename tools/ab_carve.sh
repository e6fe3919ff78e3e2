#!/bin/bash
# A/B of carve kernel variants selected by env vars: parity subset + bench (interleaved, 2 rounds)
# + ncu cycles per variant.  Usage: gpurun -- bash tools/ab_carve.sh "TCB_CARVE_SW=1" "TCB_CARVE_SW=2"
mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "carve" 2>&1 | tail -1 | sed "s/^/[$v] parity: /"
done
for r in 1 2; do
  for v in "$@"; do
    env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$v] round $r: layer', d['value'], 'carve', d['kernels_ms']['carve_fwd'], 'clk', d['clocks']['sm_mhz'], 'TF', d['kept_block_tflops'])"
  done
done
for v in "$@"; do
  env $v timeout 600 ncu --metrics sm__cycles_elapsed.avg,gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -E "sm__cycles|gpu__time|gpc__cycles|tensor_cycles|pipe_xu|dram__bytes" | sed "s/^/[$v] /"
done
