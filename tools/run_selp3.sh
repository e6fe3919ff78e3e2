timeout 600 python -m pytest tests -x -q -m gpu -k "select or mask or criterion_05 or properties or fullsize or toy or cli" 2>&1 | tail -1
cp paper_2505_16864_b200/_lib/libtcb200.so /tmp/lib_new.so
for v in new old new old; do
  if [ $v = new ]; then cp /tmp/lib_new.so paper_2505_16864_b200/_lib/libtcb200.so; else cp tools/_variant/libtcb200.so paper_2505_16864_b200/_lib/libtcb200.so; fi
  echo "== $v"; timeout 300 python tools/mask_time.py 2>&1 | tail -4
done
cp /tmp/lib_new.so paper_2505_16864_b200/_lib/libtcb200.so
