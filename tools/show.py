"""Print compact summaries of bench JSON lines: it/s, dominant kernel, per-kernel us."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d.get("roofline") or {}
    km = {k: round(v * 1e3, 1) for k, v in (r.get("kernel_ms") or {}).items()}
    e2e = d.get("e2e") or {}
    print(f, round(d.get("iters_per_s", 0), 1), r.get("kernel"), r.get("frac") and round(r["frac"], 3),
          km, e2e.get("seconds_per_step") and round(e2e["seconds_per_step"] * 1e3, 2))
