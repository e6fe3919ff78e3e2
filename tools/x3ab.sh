# fp32 (k_carve_x3) C2 carve time: this tree vs a previous build copied into ab_old/ (git-ignored)
for r in 1 2; do for tree in ab_old .; do
 (cd $tree && timeout 300 python -c "
import bench_suite as b; r=b.c2_fp32_record(); print('$tree', r['carve_ms'], r['fp32_tflops'])" 2>&1 | tail -1)
done; done
