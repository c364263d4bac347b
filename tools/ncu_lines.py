"""Per-CUDA-source-line instruction / stall-sample totals of one kernel in an ncu report.

    python tools/ncu_lines.py rep.ncu-rep KERNEL_REGEX NPOINTS [TOP]
"""
import csv
import subprocess
import sys

rep, kern, npts = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern, "--launch-count", "1"], capture_output=True, text=True).stdout
fname = "?"
hdr = None
rows = []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or len(r) < 8:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")])
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    rows.append((fname, int(r[0]), r[1].strip()[:70], ie, smp))
tot_i = sum(x[3] for x in rows) or 1
tot_s = sum(x[4] for x in rows) or 1
print(f"{kern}: {tot_i / npts * 32:.1f} thread-instr/pt, {tot_s} samples")
for f, ln, src, ie, smp in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{f}:{ln:4d} {ie / npts * 32:7.1f} instr/pt {100 * smp / tot_s:5.1f}% samp | {src}")
