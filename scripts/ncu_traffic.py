"""Summarise an ncu report: per-kernel duration and DRAM bytes, and per-stage traffic of the bench's
dominant stage (written to profiles/ncu_traffic_<config>.json for bench.py's roofline.traffic)."""
import csv
import json
import subprocess
import sys

STAGE = {
    "range": ["k_range"],
    "histogram": ["k_hist_u16", "k_hist_f32"],
    "threshold": ["k_threshold"],
    "morph": ["k_binarize", "k_open3d_reg", "k_open2d", "k_open3d"],
    "label": ["k_extract_runs", "k_union_local", "k_union_cross", "k_flatten_sizes", "k_root_flags", "k_table",
              "k_clear_dropped", "k_runs_total", "k_table_total"],
    "extract": ["k_extract_count", "k_extract"],
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    res = []
    for v in r[2:]:
        d = dict(zip(h, v))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("roix::", "").split("<")[0]
        res.append({"kernel": name, "ms": float(d.get("gpu__time_duration.sum", "nan")) / 1e6 if False else
                    float(d.get("gpu__time_duration.sum", "nan")),
                    "dram_read": float(d.get("dram__bytes_read.sum", "nan")),
                    "dram_write": float(d.get("dram__bytes_write.sum", "nan")),
                    "units": (r[1][h.index("gpu__time_duration.sum")], r[1][h.index("dram__bytes_read.sum")])})
    return res


def main(rep, config, out):
    rs = rows(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    per = {}
    for r in rs:
        f = scale.get(r["units"][1], 1)
        per.setdefault(r["kernel"], []).append((r["dram_read"] + r["dram_write"]) * f)
    stages = {}
    for st, ks in STAGE.items():
        b = sum(sum(per[k]) / len(per[k]) for k in ks if k in per)
        if any(k in per for k in ks):
            stages[st] = b
    json.dump(stages, open(out, "w"), indent=1)
    print(json.dumps(stages))


if __name__ == "__main__":
    main(*sys.argv[1:4])
