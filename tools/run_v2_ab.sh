# two-tile carve kernel (TCB_CARVE_V2=1) vs the shipped one: parity, ncu cycles/clock, bench time
TCB_CARVE_V2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5
for v2 in 0 1; do
  TCB_CARVE_V2=$v2 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__|l1tex|dram" | sed "s/^/v2=$v2 /"
done
for rep in 1 2; do for v2 in 0 1; do
  TCB_CARVE_V2=$v2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v2=$v2', d['ms_per_step'], d.get('kernels_ms'), d['clocks'])"
done; done
