timeout 300 python -m pytest tests -m gpu -x -q -k "select or pool or toy or mask or cli or relevance" 2>&1 | tail -1
for s in 1 0; do echo -n "simt=$s "; TCB_SCORES_SIMT=$s timeout 200 python bench.py --no-cpu --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms'])"; done
