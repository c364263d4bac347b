"""Summarise an ncu --page source --csv (SASS) dump: per-region instruction counts and stall samples.

    ncu -i rep --page source --csv -k regex:K --print-source sass > /tmp/src.csv
    python tools/ncu_source.py /tmp/src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = []
for r in rows[hdr_i + 1:]:
    if r and r[0] in ("Address", "Kernel Name"):
        break  # first kernel instance only
    if len(r) == len(hdr):
        data.append(r)
ci = {h: i for i, h in enumerate(hdr)}
tot_s = sum(float(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
tot_i = sum(float(r[ci["Instructions Executed"]] or 0) for r in data)
print(f"instructions={len(data)} samples={tot_s:.0f} warp_inst={tot_i:.3e}")
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and "(" not in h]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
# contiguous hot regions: cumulative over address order
acc_i = acc_s = 0.0
for k, r in enumerate(data):
    s = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    n = float(r[ci["Instructions Executed"]] or 0)
    acc_i += n
    acc_s += s
    if (k % 64) == 63:
        print(f"[{k-63:5d}..{k:5d}] {data[k-63][0][-5:]}  inst {acc_i/tot_i*100:5.1f}%  samples {acc_s/tot_s*100:5.1f}%")
        acc_i = acc_s = 0.0
print("--- top instructions by samples")
for r in sorted(data, key=lambda r: -float(r[ci["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print(f"{r[0][-5:]} {float(r[ci['Warp Stall Sampling (All Samples)']] or 0)/tot_s*100:5.2f}% "
          f"exec {float(r[ci['Instructions Executed']] or 0):.2e} thr {r[ci['Avg. Threads Executed']]:>5} {r[1].strip()[:60]}")
print("--- stall reasons per 64-instruction block (share of that block's samples)")
scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for k0 in range(0, len(data), 64):
    blk = data[k0:k0 + 64]
    tot = sum(float(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in blk)
    if tot / tot_s < 0.01:
        continue
    sums = {c: sum(float(r[ci[c]] or 0) for r in blk) for c in scols}
    top3 = sorted(sums.items(), key=lambda kv: -kv[1])[:4]
    print(f"[{k0:5d}] {tot/tot_s*100:5.1f}%  " + "  ".join(f"{c[6:]}={v/tot*100:.0f}%" for c, v in top3))
