"""Per source line: warp-instructions executed split into FP64 / other (needs -lineinfo).
usage: ncu_lines_inst.py <rep> <kernel-regex> <so> [top] [paths*steps/32 normaliser]"""
import collections, csv, glob, os, re, subprocess, sys, tempfile
rep, kern, so = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
norm = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
kname, hdr, rows = None, None, []
for l in out:
    r = next(csv.reader([l]))
    if r and r[0] == "Kernel Name":
        if kname is not None: break
        kname = r[1]; continue
    if r and r[0] == "Address": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        rows.append((int(d["Address"], 16), int(d["Instructions Executed"] or 0), d["Source"].strip()))
base = rows[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
m = re.search(r"heston_(pass\d)_kernel<(double|float), (?:\(int\))?(\d+), (?:\(bool\))?(\d)>", kname)
want = f"heston_{m.group(1)}_kernelI{m.group(2)[0]}Li{m.group(3)}ELb{m.group(4)}E" if m else kern
lines = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
    cur_fn = cur_line = None
    for l in dis.splitlines():
        if l.startswith(".text.") and l.rstrip().endswith(":"): cur_fn = l; continue
        if cur_fn is None or want not in cur_fn: continue
        mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if mm: cur_line = (os.path.basename(mm.group(1)), int(mm.group(2))); continue
        ma = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if ma and cur_line: lines[int(ma.group(1), 16)] = cur_line
fp = collections.Counter(); oth = collections.Counter(); ops = collections.defaultdict(collections.Counter)
for addr, n, src in rows:
    key = lines.get(addr - base, ("?", 0))
    mo = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
    op = mo.group(2) if mo else "?"
    if op in ("DADD", "DMUL", "DFMA"): fp[key] += n
    else: oth[key] += n; ops[key][op] += n
tf, to = sum(fp.values()), sum(oth.values())
print(f"{kname}\n  fp64 {tf/norm:.1f}  other {to/norm:.1f}  (per normaliser unit)")
for key, n in oth.most_common(top):
    top_ops = ", ".join(f"{o}:{c/norm:.1f}" for o, c in ops[key].most_common(5))
    print(f"other {n/norm:7.2f} fp64 {fp[key]/norm:7.2f}  {key[0]}:{key[1]:<4d} {top_ops}")
