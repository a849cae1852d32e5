export WH_DIAG_LIB=1
for dbg in 0 6; do
  echo "=== c4h256 tf32 dbg=$dbg  (mma: acc_empty slot = issue blocks, b_full slot = commits)"
  WH_UMMA_DBG=$dbg WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 300 python tools/prof_roles.py --config c4h256 2>&1 | tail -n 5 | grep -E "mma|converter"
done
