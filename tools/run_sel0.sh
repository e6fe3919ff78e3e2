timeout 600 ncu --set full --import-source on -k "regex:k_select" -s 2 -c 1 -f -o gpurun_out/sel0_full python tools/prof_select_p.py 0.0 > /dev/null 2>&1
