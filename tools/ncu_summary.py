"""Key metrics of ncu --set full reports -> one CSV (run where the .ncu-rep files are; the
reports themselves are too large to bring back).  usage: python tools/ncu_summary.py OUT.csv REP..."""
import csv
import io
import os
import re
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "gpc__cycles_elapsed.max", "gpc__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
    "launch__block_size", "launch__cluster_dim_x",
]
STALL = re.compile(r"^smsp__average_warp_latency_issue_stalled_(\w+)\.ratio$|"
                   r"^smsp__pcsamp_warps_issue_stalled_(\w+)$")


def rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    return r[0], r[1], r[2:]


out = sys.argv[1]
lines = [["capture", "kernel", "metric", "value", "unit"]]
for rep in sys.argv[2:]:
    name = os.path.basename(rep).replace(".ncu-rep", "")
    try:
        h, u, vals = rows(rep)
    except Exception as e:  # noqa: BLE001
        lines.append([name, "", "error", str(e)[:100], ""])
        continue
    ik = h.index("Kernel Name") if "Kernel Name" in h else None
    for v in vals:
        kern = v[ik][:60] if ik is not None else ""
        for k in WANT:
            if k in h:
                lines.append([name, kern, k, v[h.index(k)], u[h.index(k)]])
        # the largest stall reasons (pc sampling)
        st = []
        for i, k in enumerate(h):
            m = STALL.match(k)
            if m and m.group(2):
                try:
                    st.append((float(v[i].replace(",", "")), m.group(2)))
                except ValueError:
                    pass
        for val, nm in sorted(st, reverse=True)[:6]:
            lines.append([name, kern, f"stall_samples.{nm}", f"{val:.0f}", ""])
with open(out, "w", newline="") as f:
    csv.writer(f).writerows(lines)
print(f"{out}: {len(lines) - 1} rows")
