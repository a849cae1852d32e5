"""Print the UMMA plan shape of configs (diagnostics build: WH_DIAG_LIB=1 WH_UMMA_VERBOSE=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

for cfg in sys.argv[1:]:
    w = bench.workload(cfg)
    print(cfg, flush=True)
    plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"],
                       output=w["output"], norm=w["norm"], max_clips=4, engine="umma")
    plan.close()
