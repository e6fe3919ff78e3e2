# ncu --set full of the three mask-path kernels of one C2 layer (pool, DMMA scores, select)
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pool|k_scores_dmma|k_select" -s 6 -c 3 -f -o gpurun_out/mask_end python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/mask_end.log 2>&1
