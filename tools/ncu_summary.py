"""Summarise ncu artefacts into profiles/: a --set full report (SOL, memory, occupancy, stalls, top
source lines) or a gpu__time_duration launch list (per-kernel launches, time, share).

  python tools/ncu_summary.py full <report.ncu-rep> <out.json> [note]
  python tools/ncu_summary.py launches <launches.csv> <out.json> [note]
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__cycles_elapsed.avg.per_second"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def full(rep, note):
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    out = {"report": rep, "note": note, "kernel": vals[h.index("Kernel Name")][:120], "metrics": {}}
    for k in KEYS:
        if k in h:
            out["metrics"][k] = f"{vals[h.index(k)]} {units[h.index(k)]}".strip()
    # stall reasons and top source lines
    src = list(csv.reader(ncu("-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass").splitlines()))
    try:
        hdr = next(r for r in src if "Warp Stall Sampling (All Samples)" in r)
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
        agg, reasons, cur = collections.Counter(), collections.Counter(), None
        for r in src[src.index(hdr) + 1:]:
            if len(r) <= iS:
                continue
            if r[0].strip().isdigit():
                cur = (int(r[0]), r[1].strip()[:110])
                continue
            try:
                agg[cur] += float(r[iS] or 0)
                for i in cols:
                    if r[i]:
                        reasons[hdr[i]] += float(r[i])
            except ValueError:
                pass
        tot, rt = sum(agg.values()) or 1, sum(reasons.values()) or 1
        out["stall_reasons_pct"] = {k[6:]: round(100 * v / rt, 1) for k, v in reasons.most_common(8)}
        out["top_lines_pct"] = [[round(100 * v / tot, 1), f"L{k[0]}", k[1]] for k, v in agg.most_common(15) if k]
    except StopIteration:
        pass
    return out


def launches(path, note):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    iK, iV = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        k = r[iK].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[iV].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    return {"source": path, "note": note, "total_ms": tot, "n_launches": sum(v[0] for v in agg.values()),
            "kernels": {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
                        for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    res = full(src, note) if mode == "full" else launches(src, note)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
