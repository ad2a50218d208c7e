"""Per-source-line stall / instruction shares of one kernel in an ncu report: maps the SASS page of
`ncu -i REP --page source --csv --print-source sass` to source lines via `nvdisasm -g` of a cubin
built from the same sources. usage: ncu_lines.py sass.csv kernel.sass [top]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iA, iS = hdr.index("Address"), hdr.index("Source")
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
a0 = int(data[0][iA], 16)
prof = {}
for r in data:
    try:
        prof[int(r[iA], 16) - a0] = (int(r[iW]), int(r[iE]), r[iS])
    except ValueError:
        pass
cur, off2line = None, {}
for l in open(sys.argv[2]).read().split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg, agge = collections.Counter(), collections.Counter()
for off, (w, e, _) in prof.items():
    agg[off2line.get(off)] += w
    agge[off2line.get(off)] += e
tw, te = sum(agg.values()), sum(agge.values())
for k, v in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print("%5.1f%% stall  %5.1f%% inst  %s" % (100 * v / tw, 100 * agge[k] / te, k))
