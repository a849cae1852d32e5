for tf in 1 0; do
  WH_UMMA_PSTREAM=1 WH_UMMA_TF32=$tf timeout 600 python tools/tf32_check.py all 2>&1 | tail -n 12
done
timeout 300 python tools/tf32_check.py time 2>&1 | tail -n 3
