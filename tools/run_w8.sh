# A/B: shipped 2-CTA half-step kernel (impl 0) vs 1-CTA/SM Q-in-TMEM 8-softmax-warp kernel (impl 3)
TCB_CARVE_IMPL=3 timeout 300 python -m pytest tests -m gpu -x -q -k "carve or fullsize or acceptance or token_major or smoke" 2>&1 | tail -1
for impl in 0 3; do
  TCB_CARVE_IMPL=$impl timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k "regex:k_carve" -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__" | sed "s/^/impl=$impl /"
  echo -n "impl=$impl bench "; TCB_CARVE_IMPL=$impl timeout 200 python bench.py --no-cpu --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms']['carve_fwd'], d['clocks'])"
done
