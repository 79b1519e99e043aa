"""One line per bench JSON: step ms, step roofline fraction, stage times, parity."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).readline())
    except Exception as e:   # noqa: BLE001
        print(f, "unreadable", e)
        continue
    p = d.get("parity", {})
    print("%-28s %7.2f ms  frac %.3f  %s  parity %s" % (
        f.split("/")[-2] + "/" + f.split("/")[-1], d["ms_per_step"], d["step_roofline"]["frac"],
        {k: round(v, 2) for k, v in d["stage_ms"].items() if k not in ("setup", "threshold")},
        p.get("all") if isinstance(p, dict) else p))
