export WH_DIAG_LIB=1
for cg1 in 1; do
  for tf in 1 0; do
    echo "=== CG1 tf32=$tf"
    WH_UMMA_CG1=1 WH_UMMA_PSTREAM=1 WH_UMMA_TF32=$tf timeout 600 python tools/tf32_check.py time c4h256 c4h1024 2>&1 | tail -n 3
    WH_UMMA_CG1=1 WH_UMMA_PSTREAM=1 WH_UMMA_TF32=$tf WH_UMMA_VERBOSE=1 timeout 300 python tools/prof_roles.py --config c4h256 2>&1 | tail -n 6
  done
done
echo "=== CG1 rows-of-128 c4h256, c4h64"
WH_UMMA_CG1=1 timeout 600 python tools/tf32_check.py time c4h256 c4h64 2>&1 | tail -n 3
WH_UMMA_CG1=1 WH_UMMA_VERBOSE=1 timeout 300 python tools/prof_roles.py --config c4h64 2>&1 | tail -n 6
