TCB_CARVE_EMU=13 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for emu in 0 12 13 14 0 13; do
  TCB_CARVE_EMU=$emu timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__" | sed "s/^/emu=$emu /"
done
for rep in 1 2; do for emu in 0 13; do
  TCB_CARVE_EMU=$emu timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('emu=$emu', d['ms_per_step'], d['kernels_ms']['carve_fwd'], d['clocks'])"
done; done
