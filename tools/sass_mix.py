"""Per-opcode executed warp-instruction mix (and stall samples) of each kernel
in an ncu `--page source --print-source sass --csv` export (gzipped or not).
usage: sass_mix.py export.csv[.gz] [warp_units_divisor] [top]"""
import collections, csv, gzip, io, re, sys

path = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
f = io.TextIOWrapper(gzip.open(path), "utf-8") if path.endswith(".gz") else open(path)
kern, hdr, ops = None, None, collections.OrderedDict()
for row in csv.reader(f):
    if row and row[0] == "Kernel Name":
        kern = row[1]
        ops[kern] = collections.defaultdict(lambda: [0, 0])
        hdr = None
        continue
    if row and row[0] == "Address":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if not hdr or not row:
        continue
    src = row[hdr["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9_]+)*)", src)
    if not m:
        continue
    op = m.group(2).split(".")[0]
    ex = float(row[hdr["Instructions Executed"]] or 0)
    st = float(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    ops[kern][op][0] += ex
    ops[kern][op][1] += st
for k, d in ops.items():
    tot = sum(v[0] for v in d.values())
    sst = sum(v[1] for v in d.values()) or 1
    print(f"== {k[:100]}\n   total warp-inst {tot:.4g} ({tot / div:.1f} per unit)")
    for op, (ex, st) in sorted(d.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"   {op:10s} {ex / div:10.2f} {100 * ex / tot:6.2f}%   stall-samples {100 * st / sst:5.1f}%")
