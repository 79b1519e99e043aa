"""Per-stage DRAM traffic of one bench step from an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): writes profiles/ncu_traffic_<config>.json, read by
bench.py for roofline.traffic (bytes per launch of the dominant stage).

    python scripts/ncu_traffic.py gpurun_out/launches_C2.csv C2
"""
import csv
import json
import os
import sys

# kernels of each pipeline stage (one C-ABI call each; see paper_2602_15917_b200/pipeline.py)
STAGE = {
    "range": ["k_range"],
    "background": ["k_background_vec", "k_background_scalar"],
    "setup": ["k_hist_clear"],
    "histogram": ["k_hist_u16", "k_hist_u16_rw", "k_hist_f32", "k_hist_u16_frames"],
    "threshold": ["k_threshold", "k_threshold_frames"],
    "morph": ["k_binarize", "k_open3d_reg", "k_open3d_rows", "k_open2d", "k_open2d_w"],
    "label": ["k_scan_dlb", "k_runs_total", "k_runs_slots", "k_extract_runs", "k_extract_runs_rows", "k_union_local", "k_union_cross", "k_resolve_broots",
              "k_flatten_sizes", "k_largest_init", "k_largest", "k_root_flags", "k_table", "k_table_total", "k_clear_dropped", "k_table_clear"],
    "extract": ["k_extract_count", "k_extract", "k_extract_seg", "k_extract_total", "k_ck_count", "k_ck_extract",
                "k_ck_total", "k_kept_len", "k_rx_map", "k_rx_extract", "k_rx_runs", "k_gather_total"],
}


def steps(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    data, order = {}, []
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("roix::", "").split("<")[0].strip()
        k = (int(d["ID"]), name)
        if k not in data:
            order.append(k)
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        data.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
    starts = [i for i, k in enumerate(order) if k[1] == "k_scalars_init"]
    return data, order, starts


def main(path, config, out_dir="profiles"):
    data, order, starts = steps(path)
    s0 = starts[-1]                          # the last step of the run, up to its extract's total
    ends = [i for i in range(s0, len(order)) if order[i][1] in ("k_extract_total", "k_ck_total", "k_gather_total")]
    s1 = ends[0] + 1 if ends else len(order)
    kern = order[s0:s1]
    # the scan kernel appears in label and extract: attribute by position (label precedes extract)
    res, stage_of = {}, {}
    cur = None
    for k in kern:
        for st, names in STAGE.items():
            if k[1] in names and not (k[1] == "k_scan_dlb" and cur == "extract") and \
                    not (k[1] == "k_gather_total" and cur is None):
                cur = st
                break
        stage_of[k] = cur
    for k in kern:
        st = stage_of[k]
        if st is None:
            continue
        m = data[k]
        res.setdefault(st, {"dram_bytes": 0.0, "ns": 0.0, "kernels": []})
        res[st]["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        res[st]["ns"] += m.get("gpu__time_duration.sum", 0)
        res[st]["kernels"].append(k[1])
    os.makedirs(out_dir, exist_ok=True)
    dst = os.path.join(out_dir, "ncu_traffic_%s.json" % config)
    json.dump({"source": os.path.basename(path), "stages": res}, open(dst, "w"), indent=1)
    print(json.dumps({k: (round(v["dram_bytes"] / 1e6, 1), round(v["ns"] / 1e3, 1)) for k, v in res.items()}))


if __name__ == "__main__":
    main(*sys.argv[1:])
