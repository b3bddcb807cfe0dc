"""Summarise one kernel of an `ncu --page raw --csv` export into the fields of
profiles/ncu_summary.json: tools/ncu_summarize.py RAW.csv [algorithmic_bytes design_bytes]."""
import csv
import json
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ns": 1e-3, "ms": 1e3}


def summarize(path, alg=None, des=None):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(k, scale=True):
        i = hdr.index(k)
        v = float(vals[i].replace(",", ""))
        return v * SCALE.get(units[i], 1.0) if scale else v

    out = {
        "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
        "duration_us": get("gpu__time_duration.sum"),
        "dram_read_bytes": get("dram__bytes_read.sum"),
        "dram_write_bytes": get("dram__bytes_write.sum"),
        "ipc": get("sm__inst_executed.avg.per_cycle_active"),
        "warps_per_scheduler": get("smsp__warps_active.avg.per_cycle_active"),
        "eligible_warps_per_scheduler": get("smsp__warps_eligible.avg.per_cycle_active"),
        "issue_active_per_scheduler": get("smsp__issue_active.avg.per_cycle_active"),
        "registers": get("launch__registers_per_thread"),
        "warp_instructions": get("smsp__inst_executed.sum"),
        "fma_pipe_active_pct": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    }
    out["dram_bytes_per_launch"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    if alg:
        out["algorithmic_bytes_per_launch"] = alg
    if des:
        out["design_bytes_per_launch"] = des
    pre, post = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    out["stalls_per_issue"] = {k[len(pre):-len(post)]: round(get(k), 3) for k in hdr
                               if k.startswith(pre) and k.endswith(post) and get(k) >= 0.05}
    return out


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[2:4]] + [None, None]
    print(json.dumps(summarize(sys.argv[1], a[0], a[1]), indent=1))
