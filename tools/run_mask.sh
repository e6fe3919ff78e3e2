# mask-path kernels: parity tests, bench timings, ncu source-level capture of k_select
timeout 300 python -m pytest tests -m gpu -x -q -k "pool or select or toy or layer" 2>&1 | tail -1
timeout 200 python bench.py --no-cpu --no-e2e --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms'], d['clocks'])"
timeout 300 ncu --set full --import-source on --clock-control none -k "regex:k_select|k_scores" -s 6 -c 2 -o gpurun_out/mask_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out/
