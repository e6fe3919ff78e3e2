#!/bin/bash
# One gpurun call: tests + profiles.  Usage: gpurun -- bash tools/gpu_round.sh <what...>
# (what: tests ref fullsize hbm hbmncu bench benchq launches carvencu sanitize)
set -o pipefail
mkdir -p gpurun_out
for w in "$@"; do
  case "$w" in
    tests)     python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/gpu_tests.log; tail -1 gpurun_out/gpu_tests.log ;;
    ref)       python -m pytest tests/ref_suite -q -m gpu -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/ref_suite.log; tail -1 gpurun_out/ref_suite.log ;;
    fullsize)  rm -f gpurun_out/fullsize_parity.jsonl; TCB_REPORT_DIR=gpurun_out python -m pytest tests/test_gpu_fullsize_configs.py -q -m gpu -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/fullsize.log; tail -1 gpurun_out/fullsize.log ;;
    hbm)       python tools/prof_hbm.py --out gpurun_out/hbm_kernels.json > /dev/null 2>gpurun_out/hbm.err; tail -2 gpurun_out/hbm.err ;;
    hbmncu)    ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_upsample|k_rope|k_curve|k_adjacency|k_pool' -f -o gpurun_out/hbm python tools/prof_hbm.py --ncu > gpurun_out/hbmncu.log 2>&1; tail -2 gpurun_out/hbmncu.log ;;
    bench)     python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json ;;
    benchq)    python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    launches)  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; wc -l gpurun_out/launches.csv ;;
    carvencu)  ncu --set full --clock-control none --import-source on -k regex:k_carve_tc -c 1 -f -o gpurun_out/carve python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/carvencu.log 2>&1; tail -2 gpurun_out/carvencu.log ;;
    sanitize)  for t in memcheck racecheck synccheck; do timeout 1500 compute-sanitizer --tool $t --print-limit 5 python -m pytest tests/test_gpu_parity.py tests/test_gpu_carve_split.py tests/test_gpu_select_p0.py tests/test_gpu_select_cut.py -q -p no:cacheprovider -x -k "split or extremes or fuzz or select or 931 or 256" 2>&1 | grep -E "SUMMARY|passed|failed" | sed "s/^/[$t] /"; done ;;
    *) echo "unknown $w" ;;
  esac
done
