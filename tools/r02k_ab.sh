for c in c2 c3 c4h64 c4h16 c5; do
  timeout 300 python tools/ab.py paper_2408_14302_b200/libwavehop_b200.so $c 2>&1 | tail -n 1
done
