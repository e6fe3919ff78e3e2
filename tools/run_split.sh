TCB_CARVE_SPLIT=1 timeout 300 python -m pytest tests -m gpu -x -q -k "carve" 2>&1 | tail -1
for sp in 0 1; do
  TCB_CARVE_SPLIT=$sp timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_carve_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "gpu__|sm__|gpc__|dram__|lts__" | sed "s/^/split=$sp /"
  echo -n "split=$sp bench "; TCB_CARVE_SPLIT=$sp timeout 200 python bench.py --no-cpu --no-e2e --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms']['carve_fwd'], d['clocks'])"
done
