"""Summarise ncu DRAM traffic of every k_pcg_r launch of one C2 step against the device-counted
algorithmic bytes (tools/pcg_traffic.py output) → JSON (bench.py reads it for roofline.traffic)."""
import csv, json, re, sys
csvf, logf, out = sys.argv[1:4]
rows = [r for r in csv.reader(open(csvf)) if len(r) > 10]
h, rows = rows[0], rows[1:]
iK, iN, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows:
    if not r[iK].startswith("k_pcg_r"):
        continue
    per.setdefault(r[iID], {})[r[iN]] = float(r[iV].replace(",", ""))
unit = {"dram__bytes_read.sum": 1.0, "dram__bytes_write.sum": 1.0}
alg = json.loads(re.search(r"ALG (\{.*\})", open(logf).read()).group(1))
n = len(per)
dram = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
ms = sum(v.get("gpu__time_duration.sum", 0) for v in per.values()) / 1e6
res = {"kernel": "k_pcg_r", "launches": n, "dram_bytes_per_launch": dram / max(n, 1),
       "alg_bytes_per_launch": alg["alg_bytes_step"] / max(n, 1), "traffic_over_alg": dram / max(alg["alg_bytes_step"], 1),
       "ncu_ms_total": ms, "pcg_iters_step": alg["pcg_iters_step"], "envs": alg["envs"], "step": alg["step"],
       "capture": "ncu --profile-from-start off -k regex:k_pcg_r --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                  "gpu__time_duration.sum over one C2 step (tools/pcg_traffic.py 1024 12); units: bytes, ns",
       "note": "env-resident PCG: the condensed operator is staged into shared memory once per launch, so DRAM "
               "traffic per launch is far below the per-iteration streaming (algorithmic) bytes"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
