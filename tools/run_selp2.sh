timeout 300 ncu --metrics gpu__time_duration.sum --csv -s 12 python tools/prof_select_p.py 0.3 > gpurun_out/selp_launch.csv 2>&1
timeout 600 ncu --set full --import-source on -k "regex:k_select" -s 4 -c 2 -f -o gpurun_out/selp_full python tools/prof_select_p.py 0.3 > /dev/null 2>&1
