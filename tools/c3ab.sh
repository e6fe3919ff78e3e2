# C3 / C2 carve timing of this tree vs the round-1 build copied into ab_r01/ (git-ignored)
for r in 1 2; do
for tree in . ab_r01; do
 (cd $tree && timeout 300 python -c "
import bench_suite as b
c3=b.layer_record('C3',(21,30,52),0,40,0.08); c2=b.layer_record('C2',(33,45,80),256,24,0.08)
print('$tree', 'C3 carve', c3['carve_ms'], 'mask', c3['mask_ms'], '| C2 carve', c2['carve_ms'], 'mask', c2['mask_ms'])" 2>&1 | tail -1)
done; done
