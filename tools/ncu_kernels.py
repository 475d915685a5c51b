"""Per-launch summary of an `ncu --set full` capture (any kernels): duration,
grid, registers, DRAM bytes and throughput, FP64 / DMMA pipe use, SM
throughput and the top warp-stall reasons (sampled).
    python tools/ncu_kernels.py REP.ncu-rep --what "..." > profiles/r02/X.json"""
import argparse
import csv
import io
import json
import subprocess

M = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "registers": ("launch__registers_per_thread", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "fp64_pipe_pct_active": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "dmma_pipe_pct_active": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
}


def num(v, unit):
    v = float(v.replace(",", ""))
    u = (unit or "").lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return v * scale.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--what", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = {"capture": a.rep.split("/")[-1], "what": a.what, "launches": []}
    for r in rows[2:]:
        rec = {"kernel": r[idx["Kernel Name"]][:90]}
        for k, (m, _) in M.items():
            if m in idx and r[idx[m]] not in ("", "n/a"):
                val = num(r[idx[m]], units[idx[m]])
                if k == "duration_us" and units[idx[m]].lower() == "nsecond":
                    val = float(r[idx[m]].replace(",", "")) / 1e3
                rec[k] = round(val, 3) if isinstance(val, float) else val
        st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[i].replace(",", "") or 0)
              for h, i in idx.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
        tot = sum(st.values()) or 1.0
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:4]}
        res["launches"].append(rec)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
