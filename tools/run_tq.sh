# A/B of the carve kernels (round-1 tc vs Q-in-TMEM tq) with pipeline-ceiling knobs
for impl in 0 1; do
  TCB_CARVE_IMPL=$impl timeout 300 python -m pytest tests -m gpu -x -q -k "carve" 2>&1 | tail -1
done
for impl in 0 1; do for dbg in 0 1 2 3; do
  echo -n "impl=$impl dbg=$dbg "; TCB_CARVE_IMPL=$impl TCB_CARVE_DEBUG=$dbg timeout 200 python bench.py --no-cpu --no-e2e --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms']['carve_fwd'], d['clocks'])"
done; done
for emu in 2 3; do for impl in 0 1; do echo -n "impl=$impl emu=$emu "; TCB_CARVE_IMPL=$impl TCB_CARVE_EMU=$emu timeout 200 python bench.py --no-cpu --no-e2e --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms']['carve_fwd'], d['clocks'])"; done; done
