"""Summarise an ncu report: top CUDA source lines by warp-stall samples and overall stall reasons."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
iS = hdr.index("Warp Stall Sampling (All Samples)")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg, reasons, cur = collections.Counter(), collections.Counter(), None
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= iS:
        continue
    if r[0].strip().isdigit():
        cur = (int(r[0]), r[1].strip()[:100])
        continue
    try:
        agg[cur] += float(r[iS] or 0)
        for i in cols:
            if r[i]:
                reasons[hdr[i]] += float(r[i])
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {v / sum(reasons.values()) * 100:.0f}%" for k, v in reasons.most_common(6)))
for k, v in agg.most_common(n):
    print(f"{v / tot * 100:5.1f}%  L{k[0] if k else '?'}  {k[1] if k else ''}")
