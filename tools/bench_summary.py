"""Print the key numbers of bench JSON lines (files given on the command line)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    sh = (d.get("variants") or {}).get("shared_maps") or {}
    print(f, f"ms/apply {d['ms_per_step']:.4f}", f"roof {d['roofline']['bound']} {d['roofline']['frac']:.3f}",
          "gmres", {k: d["gmres"][k] for k in ("time_to_solution_s", "iterations")} if d.get("gmres") else None,
          "| shared", f"{sh.get('ms_per_apply', 0):.4f} ms", sh.get("roofline", {}).get("frac"),
          {k: sh["gmres"][k] for k in ("time_to_solution_s", "iterations")} if sh.get("gmres") else None)
