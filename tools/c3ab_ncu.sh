# ncu counters of the C2 carve launch: this tree vs ab_r01/ (round-1 build)
for tree in . ab_r01; do
 (cd $tree && timeout 600 ncu --metrics sm__cycles_elapsed.avg,smsp__inst_executed.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed_pipe_xu.sum,gpc__cycles_elapsed.avg.per_second,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum -k regex:k_carve_tc -c 1 --clock-control none python -c "
import bench_suite as b
L=b.Layer((33,45,80),256,24,0.08); L.mask(); L.carve()" 2>&1 | grep -E "sm__|smsp__|dram|lts|gpc|l1tex" | sed "s|^|[$tree] |")
done
