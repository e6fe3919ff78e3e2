# carve A/B under ncu: cycles and clock for TCB_CARVE_DEBUG values given as arguments
for dbg in "$@"; do
  TCB_CARVE_DEBUG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__" | sed "s/^/dbg=$dbg /"
done
