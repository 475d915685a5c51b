"""Summarise an ncu capture of the step-apply kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_step_cfg5.ncu-rep --config 5 --first-launch 20 \
        --launches-csv gpurun_out/launches_cfg5.csv --out profiles/ncu_step_kernel_cfg5.json

For each captured k_step1 launch: duration, DRAM bytes (read + write) and the
ALGORITHMIC bytes of that launch (16 (rows K + K + 2 rows) per
solve-application, summed over the step's items), so traffic / algorithmic
shows re-reads.  The launch index i maps to BSP step (i mod steps_per_apply):
forward steps, the residual (full) step, backward steps.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (r[i], units[i]) for i, h in enumerate(hdr)} for r in rows[2:]]


def step_bytes(cfgno):
    """Algorithmic bytes of every step-apply launch of one BSP apply, in launch order."""
    from oracle.lattice import Lattice, windows
    from paper_2209_10886_b200.configs import CONFIGS
    c = CONFIGS[cfgno]
    lat = Lattice(c["n1"], c["n2"])
    n = c["n"]

    def item_bytes(s, rows):
        K = len(lat.faces[s]) * n
        return 16.0 * (rows * K + K + 2 * rows)

    def nlower(s):
        return sum(1 for f, _ in lat.faces[s] if f in (0, 1))

    out = []
    lw = windows(c["n1"], c["n2"], "lower", c["blocks"])
    for t in range(1, max(hi - lo for lo, hi in lw) + 1):
        out.append(sum(item_bytes(s, (len(lat.faces[s]) - nlower(s)) * n)
                       for lo, hi in lw if t <= hi - lo for s in lat.groups.get(lo + t - 1, [])
                       if len(lat.faces[s]) > nlower(s)))
    out.append(sum(item_bytes(s, len(lat.faces[s]) * n) for s in lat.subs))
    uw = windows(c["n1"], c["n2"], "upper", c["blocks"])
    for t in range(1, max(hi - lo for lo, hi in uw) + 1):
        out.append(sum(item_bytes(s, nlower(s) * n)
                       for lo, hi in uw if t <= hi - lo for s in lat.groups.get(hi - t + 1, []) if nlower(s)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--first-launch", type=int, default=20, help="index of the first captured k_step1 launch")
    ap.add_argument("--launches-csv", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--fused", action="store_true", help="one launch = one whole BSP apply (k_bsp_fused)")
    ap.add_argument("--kernel", default="k_step1<16>")
    ap.add_argument("--alg-bytes", type=float, default=None,
                    help="algorithmic bytes of one captured launch (the map-once plan's, from the bench line's "
                         "roofline.algorithmic_bytes_per_apply); default: the per-step formula of SURVEY.md 8d")
    ap.add_argument("--bench-json", default=None, help="read --alg-bytes from this bench line")
    a = ap.parse_args()
    per_step = step_bytes(a.config)
    if a.fused:
        per_step = [sum(per_step)]
    if a.bench_json:
        with open(a.bench_json) as f:
            a.alg_bytes = json.loads(f.read().strip().splitlines()[-1])["roofline"]["algorithmic_bytes_per_apply"]
    if a.alg_bytes:
        per_step = [a.alg_bytes]
    launches = []
    for i, r in enumerate(raw_rows(a.rep)):
        idx = a.first_launch + i
        alg = per_step[idx % len(per_step)]
        dram = float(r["dram__bytes_read.sum"][0]) * (1e6 if r["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if r["dram__bytes_read.sum"][1] == "Gbyte" else 1)
        dw = float(r["dram__bytes_write.sum"][0]) * (1e6 if r["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if r["dram__bytes_write.sum"][1] == "Gbyte" else 1)
        du = r["gpu__time_duration.sum"][1]
        dur_us = float(r["gpu__time_duration.sum"][0]) * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(du, 1.0)
        launches.append({"launch_index": idx, "bsp_step": idx % len(per_step), "duration_us": dur_us,
                         "dram_read_bytes": dram, "dram_write_bytes": dw, "algorithmic_bytes": alg,
                         "traffic_over_algorithmic": (dram + dw) / alg,
                         "dram_pct_peak": float(r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
                         "registers": int(float(r["launch__registers_per_thread"][0])),
                         "grid": int(float(r["launch__grid_size"][0])),
                         "warps_active_pct": float(r["sm__warps_active.avg.pct_of_peak_sustained_active"][0])})
    summ = {"kernel": a.kernel, "config": a.config, "source": os.path.basename(a.rep),
            "note": "ncu --set full --clock-control none, cold cache, serialised replays",
            "launches": launches,
            "dram_bytes_per_launch": sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in launches) / len(launches),
            "algorithmic_bytes_per_launch": sum(x["algorithmic_bytes"] for x in launches) / len(launches),
            "traffic_over_algorithmic": sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in launches)
            / sum(x["algorithmic_bytes"] for x in launches),
            "bsp_step_algorithmic_bytes": per_step}
    if a.launches_csv and os.path.exists(a.launches_csv):
        with open(a.launches_csv) as f:
            lines = [ln for ln in f if not ln.startswith("==")]
        rows = list(csv.DictReader(io.StringIO("".join(lines))))
        tot = {}
        for r in rows:
            if r.get("Metric Name") == "gpu__time_duration.sum":
                k = r["Kernel Name"].split("(")[0]
                v = float(r["Metric Value"].replace(",", ""))
                tot[k] = tot.get(k, 0.0) + v
        s = sum(tot.values())
        summ["launch_list_share"] = {k: v / s for k, v in tot.items()} if s else {}
        summ["launch_list_count"] = len([r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"])
    with open(a.out, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps({k: v for k, v in summ.items() if k != "launches"}, indent=1))


if __name__ == "__main__":
    main()
