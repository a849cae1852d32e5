# role waits + CTA-0 timeline for c2 and c5 (diagnostics; not bench values)
for c in c2 c5; do
  timeout 120 python tools/prof_roles.py --config $c > gpurun_out/roles_$c.txt 2>&1
  timeout 120 python tools/trace_units.py --config $c > gpurun_out/trace_$c.txt 2>&1
done
WH_UMMA_VERBOSE=1 timeout 120 python tools/run_plan.py --iters 1 > gpurun_out/plan_c2.txt 2>&1
tail -n 30 gpurun_out/roles_c2.txt gpurun_out/trace_c2.txt gpurun_out/roles_c5.txt gpurun_out/trace_c5.txt gpurun_out/plan_c2.txt
