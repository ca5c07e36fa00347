"""Summarise ncu --set full captures into profiles/ (committed evidence).

    python scripts/ncu_summary.py OUT_DIR report.ncu-rep [...]

Writes OUT_DIR/<report>.txt (key metrics + top SASS stall sites) and merges
per-launch DRAM traffic into profiles/ncu_traffic.json, which bench.py reads
for roofline.traffic (keyed by kernel and config).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = (r[i], u[i])
        d["kernel"] = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        res.append(d)
    return res


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    outdir = sys.argv[1]
    os.makedirs(outdir, exist_ok=True)
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rep in sys.argv[2:]:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        lines = [f"# {name}  (ncu --set full --clock-control none; cold-cache replay)"]
        for d in raw(rep):
            lines.append(f"kernel: {d['kernel'][:110]}")
            for k in KEYS:
                if k in d:
                    lines.append(f"  {k:62s} {d[k][0]:>18s} {d[k][1]}")
            if "dram__bytes_read.sum" in d:
                b = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
                lines.append(f"  dram bytes read+write per launch: {b:.4e}")
                parts = name.split("_")          # prof_<kernel>_<cfg>
                kern = "_".join(parts[1:-1])
                cfg = parts[-1]
                traffic.setdefault(cfg, {})[kern] = {"bytes": b, "report": os.path.basename(rep)}
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(src)))
        if len(rows) > 2:
            h = rows[1]
            ix = {k: i for i, k in enumerate(h)}
            data = rows[2:]
            num = lambda x: float(x) if x not in ("", None) else 0.0  # noqa: E731
            tot = sum(num(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data) or 1.0
            stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
            agg = sorted(((sum(num(r[ix[k]]) for r in data) / tot, k) for k in stalls), reverse=True)[:8]
            lines.append("stall reasons (share of samples): " + ", ".join(f"{k[6:]} {v*100:.1f}%" for v, k in agg))
            top = sorted(data, key=lambda r: -num(r[ix["Warp Stall Sampling (All Samples)"]]))[:12]
            lines.append("top stall sites:")
            for r in top:
                lines.append(f"  {num(r[ix['Warp Stall Sampling (All Samples)']]) / tot * 100:5.1f}%  "
                             f"exec={num(r[ix['Instructions Executed']]):>10.0f}  {r[ix['Source']][:70]}")
        open(os.path.join(outdir, name + ".txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines[:22]))
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
