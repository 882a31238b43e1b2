"""Summarise the ncu DRAM traffic of every PCG launch of one lockstep step against the device-counted
algorithmic bytes (tools/pcg_traffic.py output) and merge it into profiles/r2_pcg_traffic.json under the
workload's name (bench.py reads it for roofline.traffic).

  python tools/pcg_traffic_summary.py <ncu.csv> <pcg_traffic.log> <out.json>"""
import csv, json, os, re, sys
csvf, logf, out = sys.argv[1:4]
rows = [r for r in csv.reader(open(csvf)) if len(r) > 10]
h, rows = rows[0], rows[1:]
iK, iN, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
alg = json.loads(re.search(r"ALG (\{.*\})", open(logf).read()).group(1))
kname = alg["kernel"].split(" ")[0]
per = {}
import re as _re
def _base(n):    # "void k_pcg<2>(Dev, ...)" -> "k_pcg"
    n = n.split("(")[0].strip()
    n = n.split(" ")[-1]
    return _re.sub(r"<.*>$", "", n)
for r in rows:
    if _base(r[iK]) != kname:
        continue
    per.setdefault(r[iID], {})[r[iN]] = float(r[iV].replace(",", ""))
n = len(per)
dram = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
ms = sum(v.get("gpu__time_duration.sum", 0) for v in per.values()) / 1e6
res = {"kernel": kname, "launches": n, "dram_bytes_per_launch": dram / max(n, 1),
       "alg_bytes_per_launch": alg["alg_bytes_step"] / max(n, 1), "traffic_over_alg": dram / max(alg["alg_bytes_step"], 1),
       "ncu_ms_total": ms, "pcg_iters_step": alg["pcg_iters_step"], "envs": alg["envs"], "step": alg["step"],
       "what": (f"every {kname} launch of lockstep step {alg['step']} of {alg['cfg']} x {alg['envs']} envs "
                f"(tools/pcg_traffic.py); per launch, bytes")}
allr = json.load(open(out)) if os.path.exists(out) else {}
allr[alg["cfg"]] = res
json.dump(allr, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
