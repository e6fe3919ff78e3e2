TCB_CARVE_V2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for cfg in "0 0" "1 0" "1 3" "2 0"; do set -- $cfg
  TCB_CARVE_V2=$1 TCB_CARVE_DEBUG=$2 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__" | sed "s/^/v2=$1 dbg=$2 /"
done
echo "== trace NT=1"; TCB_CARVE_V2=1 TCB_CARVE_DEBUG=8 timeout 300 python tools/carve_trace.py --dump 0 2>&1 | grep tile
for v2 in 0 1 0 1; do
  TCB_CARVE_V2=$v2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v2=$v2', d['ms_per_step'], d.get('kernels_ms'), d['clocks'])"
done
