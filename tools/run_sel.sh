timeout 300 python -m pytest tests -m gpu -x -q -k "select or pool or toy or mask or cli" 2>&1 | tail -1
timeout 200 python bench.py --no-cpu --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms'], d['clocks'])"
