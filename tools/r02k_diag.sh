# role waits + CTA-0 timelines for the large hops (both row schemes), c2 and c5 (diagnostics build)
export WH_DIAG_LIB=1
for c in c4h1024 c4h256 c4h64 c2 c5; do
  for ps in 0 1; do
    if [ $ps = 1 ] && { [ $c = c2 ] || [ $c = c5 ] || [ $c = c4h64 ]; }; then continue; fi
    echo "=== $c pstream=$ps"
    WH_UMMA_PSTREAM=$ps WH_UMMA_VERBOSE=1 timeout 300 python tools/prof_roles.py --config $c 2>&1 | tail -n 12
    WH_UMMA_PSTREAM=$ps timeout 300 python tools/trace_units.py --config $c 2>&1 | tail -n 16
  done
done
