export WH_DIAG_LIB=1
for dbg in 0 2048 32 1; do
  echo "=== c5 dbg=$dbg (2048: no store instructions; 32: TMEM loads + re-zeroing only; 1: no epilogue work)"
  WH_UMMA_DBG=$dbg timeout 300 python tools/prof_roles.py --config c5 2>&1 | tail -n 5 | grep -E "mma|epilogue"
done
