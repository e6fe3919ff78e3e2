timeout 600 python -m pytest tests -x -q -m gpu -k "select or mask or criterion_05 or properties or fullsize or toy or cli or graph" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/mask_time.py 2>&1 | tail -4; done
