"""Per-kernel time share and DRAM bytes from an ncu --metrics launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum), for the LAST step of the command: markdown table on
stdout; with --phase NAME K1,K2,.. also the summed DRAM bytes of those kernels in that step."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launches = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0].split("::")[-1])
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    launches.setdefault(key, {})[d["Metric Name"]] = v * scale
per = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (lid, name), m in launches.items():
    p = per[name]
    p[0] += 1
    p[1] += m.get("gpu__time_duration.sum", 0.0)
    p[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(p[1] for p in per.values())
print("| kernel | launches | total us | share | DRAM bytes (read+write) |")
print("|---|---|---|---|---|")
for name, (c, t, b) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print("| %s | %d | %.1f | %.1f%% | %.3g |" % (name, c, t, 100 * t / tot if tot else 0, b))
