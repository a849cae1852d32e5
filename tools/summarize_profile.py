"""Summarise a round's ncu artefacts into profiles/ (run here, no GPU needed).

usage: python tools/summarize_profile.py TAG   (reads gpurun_out/{launches,prof_umma_c2,bench}_TAG*)"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
out = "profiles"
# launch list -> per-kernel shares
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"usecond": 1e3, "msecond": 1e6}.get(r[iu], 1.0)
    a = agg.setdefault(r[ik][:70], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none): python bench.py --steps 2 --warmup 1 "
         "--no-cpu-baseline --no-e2e (c2); cold-cache serialised -- compare SHARES",
         "# per step the hot path launches exactly one kernel (wh::k_umma); the fill kernels are the bench's "
         "L2 flush, the bank builders run once at plan creation", "kernel,launches,total_ns,share"]
for k, (n, v) in agg.items():
    lines.append(f'"{k}",{n},{v:.0f},{v / tot:.3f}')
open(f"{out}/{tag}_launches_summary.csv", "w").write("\n".join(lines) + "\n")
shutil.copy(f"gpurun_out/launches_{tag}.csv", f"{out}/{tag}_launches.csv")
for c in ("c2", "c5", "ref"):
    if os.path.exists(f"gpurun_out/bench_{c}_{tag}.json"):
        shutil.copy(f"gpurun_out/bench_{c}_{tag}.json", f"{out}/{tag}_bench_{c}.json")
if os.path.exists(f"gpurun_out/bench_{tag}.json"):
    shutil.copy(f"gpurun_out/bench_{tag}.json", f"{out}/{tag}_bench_c2.json")
# full capture -> key metrics
rep = f"gpurun_out/prof_umma_c2_{tag}.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__cluster_dim_x"]
m = {}
txt = [f"# ncu --set full --clock-control none capture of wh::k_umma (BASELINE c2: 64 clips x 160000, 128 scales,",
       "# hop 64, log1p); command: ncu --set full --clock-control none --import-source on -k regex:k_umma -s 1 -c 1",
       "#   python tools/run_plan.py --iters 2   (replayed ~40x, cold cache: durations are not bench values)"]
for k in want:
    if k in hdr:
        i = hdr.index(k)
        m[k] = vals[i]
        txt.append(f"{k} = {vals[i]} {units[i]}")
open(f"{out}/{tag}_ncu_k_umma_c2.txt", "w").write("\n".join(txt) + "\n")
traffic = float(m["dram__bytes_read.sum"]) * 1e6 + float(m["dram__bytes_write.sum"]) * 1e6
tj = json.load(open(f"{out}/traffic.json")) if os.path.exists(f"{out}/traffic.json") else {}
tj["c2:umma:64"] = int(traffic)
tj["_note"] = f"dram__bytes_read.sum + dram__bytes_write.sum of one k_umma launch, ncu --set full ({out}/{tag}_ncu_k_umma_c2.txt)"
json.dump(tj, open(f"{out}/traffic.json", "w"), indent=1)
print("\n".join(lines))
print("\n".join(txt))
