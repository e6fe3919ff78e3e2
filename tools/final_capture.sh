# Round-end measurement set: bench line (with CPU baseline + e2e), reference arm, ncu launch
# list, one --set full capture of the carve kernel, and the smoke test.
set -x
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_carve_tc -s 3 -c 1 \
  -f -o gpurun_out/final_carve python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/final_carve.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
ls -la gpurun_out/
