"""Summary JSON of an ncu --set full report (per kernel: duration, DRAM bytes, issue, pipes,
shared-memory wavefronts / conflicts, registers, stall reasons) for profiles/.

    python tools/ncu_summary.py rep.ncu-rep "capture command" > profiles/NAME.json
"""
import csv
import json
import subprocess
import sys

rep, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
res = {"capture": cmd, "kernels": {}}
seen = set()
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if name in seen:
        continue  # first launch of each kernel
    seen.add(name)
    k = {}
    for w in WANT:
        if w in hdr:
            k[w] = f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip()
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") or h.startswith("smsp__pcsamp_warps_issue_stalled_"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0:
                st[h.split("stalled_")[-1]] = v
    if st:
        tot = sum(st.values())
        k["stall_share"] = {kk: round(v / tot, 4) for kk, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]}
    res["kernels"][name] = k
print(json.dumps(res, indent=1))
