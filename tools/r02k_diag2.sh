export WH_DIAG_LIB=1
for c in c4h1024; do
  for dbg in 0 16; do
    echo "=== $c tf32 dbg=$dbg"
    WH_UMMA_DBG=$dbg WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 300 python tools/prof_roles.py --config $c 2>&1 | tail -n 5
  done
done
