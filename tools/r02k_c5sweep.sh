for g in 0 16 24 32 40; do
  if [ $g = 0 ]; then echo "== default"; timeout 300 python tools/ab.py paper_2408_14302_b200/libwavehop_b200.so c5 2>&1 | tail -n 1
  else echo "== GROUP_KB=$g"; WH_UMMA_GROUP_KB=$g timeout 300 python tools/ab.py paper_2408_14302_b200/libwavehop_b200.so c5 2>&1 | tail -n 1; fi
done
for g in 16 24 32; do
  echo "== PREFER_DOUBLE GROUP_KB=$g"; WH_UMMA_PREFER_DOUBLE=1 WH_UMMA_GROUP_KB=$g timeout 300 python tools/ab.py paper_2408_14302_b200/libwavehop_b200.so c5 2>&1 | tail -n 1
done
echo "== PREFER_DOUBLE"; WH_UMMA_PREFER_DOUBLE=1 timeout 300 python tools/ab.py paper_2408_14302_b200/libwavehop_b200.so c5 2>&1 | tail -n 1
