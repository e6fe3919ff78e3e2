# split-key carve kernel (TCB_CARVE_V6=1) vs the shipped one: parity, ncu cycles/clock, bench
TCB_CARVE_V6=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -m gpu 2>&1 | tail -3
for cfg in "0 0" "1 0" "1 3" "1 2"; do set -- $cfg
  TCB_CARVE_V6=$1 TCB_CARVE_DEBUG=$2 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__" | sed "s/^/v6=$1 dbg=$2 /"
done
for v6 in 0 1 0 1; do
  TCB_CARVE_V6=$v6 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v6=$v6', d['ms_per_step'], d['kernels_ms']['carve_fwd'], d['clocks'])"
done
