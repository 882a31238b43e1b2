"""Summarise an ncu --page raw --csv export (one row per captured launch) into JSON: per launch the
grid, duration, DRAM bytes, issue/warp activity, shared-memory wavefronts and the stall mix.

  python tools/ncu_raw_summary.py <raw.csv> <out.json> <note>
"""
import csv
import json
import sys

KEYS = {"kernel": "Kernel Name", "grid": "launch__grid_size", "block": "launch__block_size",
        "regs": "launch__registers_per_thread", "duration": "gpu__time_duration.sum",
        "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smem_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smem_ld_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct", "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"}


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return v


def main(src, dst, note):
    rows = list(csv.reader(open(src)))
    h, units = rows[0], rows[1]
    out = {"source": src, "note": note, "launches": []}
    for r in rows[2:]:
        d = {}
        for k, col in KEYS.items():
            if col in h:
                i = h.index(col)
                d[k] = num(r[i]) if k != "kernel" else r[i][:80]
                if units[i] and k not in ("kernel", "grid", "block", "regs"):
                    d[k + "_unit"] = units[i]
        st = {c.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(r[i]) for i, c in enumerate(h)
              if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")}
        tot = sum(v for v in st.values() if isinstance(v, float))
        if tot:
            d["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1] if isinstance(x[1], float) else 0)[:8]}
        out["launches"].append(d)
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:4])
