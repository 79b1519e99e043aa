"""Print one step's launches (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum csv)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
h = rows[0]
data, order = {}, []
for r in rows[1:]:
    d = dict(zip(h, r))
    k = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", "").replace("roix::", "")[:34])
    if k not in data:
        order.append(k)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6}.get(d.get("Metric Unit", ""), 1)
    data.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
starts = [i for i, k in enumerate(order) if "k_scalars_init" in k[1]]
which = int(sys.argv[2]) if len(sys.argv) > 2 else -2
s0 = starts[which]
s1 = starts[which + 1] if which + 1 < len(starts) and which != -1 else len(order)
ends = [i for i in range(s0, s1) if any(t in order[i][1] for t in ("k_extract_total", "k_ck_total", "k_gather_total"))]
s1 = ends[0] + 1 if ends else s1
tot = 0
for k in order[s0:s1]:
    m = data[k]
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
    print("%4d %-34s %9.1f us  rd %9.1f MB  wr %9.1f MB  %7.2f TB/s" % (k[0], k[1], t, rd / 1e6, wr / 1e6,
                                                                       (rd + wr) / max(t, 1e-9) / 1e6))
print("total %.1f us" % tot)
