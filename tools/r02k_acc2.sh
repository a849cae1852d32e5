export WH_DIAG_LIB=1
for a2 in 1 0; do
  echo "=== acc2=$a2"
  WH_UMMA_ACC2=$a2 WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 600 python tools/tf32_check.py all 2>&1 | tail -n 8
  WH_UMMA_ACC2=$a2 WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 300 python tools/prof_roles.py --config c4h256 2>&1 | tail -n 5
done
