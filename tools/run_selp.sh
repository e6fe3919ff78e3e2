timeout 300 python -m pytest tests -m gpu -x -q -k "select or pool or toy or mask or cli or fullsize" 2>&1 | tail -1
timeout 300 python tools/prof_select_p.py 0.3
timeout 300 ncu --metrics gpu__time_duration.sum -k "regex:k_select" -s 2 -c 1 python tools/prof_select_p.py 0.3 2>&1 | grep gpu__time
timeout 300 ncu --metrics gpu__time_duration.sum -k "regex:k_select" -s 2 -c 1 python tools/prof_select_p.py 0.7 2>&1 | grep gpu__time
