export WH_DIAG_LIB=1
echo "=== TMA"
WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 600 python tools/tf32_check.py all 2>&1 | tail -n 8
WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 300 python tools/prof_roles.py --config c4h1024 2>&1 | tail -n 5
WH_UMMA_PSTREAM=1 WH_UMMA_TF32=1 timeout 300 python tools/trace_panels.py c4h1024 2>&1 | tail -n 6
