"""Attribute ncu per-SASS stall samples / executed instructions to source lines.

usage: ncu_lines.py <report.ncu-rep | source-page.csv[.gz]> <kernel-regex> <engine .so> [top]
Joins `ncu --page source --print-source sass` (per-address samples) with the
line table of `nvdisasm -g` on the cubin inside the .so (needs -lineinfo)."""
import collections, csv, glob, io, os, re, subprocess, sys, tempfile

rep, kern, so = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

if rep.endswith(".csv") or rep.endswith(".csv.gz"):  # an exported source page (gpu_profile.sh)
    import gzip
    out = (gzip.open(rep, "rt") if rep.endswith(".gz") else open(rep)).read().splitlines()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}", "--print-source", "sass"], capture_output=True,
                         text=True).stdout.splitlines()
kname = None
rows = []
hdr = None
for l in out:
    r = next(csv.reader([l]))
    if r and r[0] == "Kernel Name":
        if kname is not None:
            break  # first matching kernel only
        if re.search(kern, r[1]):
            kname = r[1]
        continue
    if kname is None:
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        rows.append((int(d["Address"], 16), int(d["Warp Stall Sampling (All Samples)"] or 0),
                     int(d["Instructions Executed"] or 0), d["Source"].strip()))
base = rows[0][0]

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
# demangled template arguments -> the mangled name's argument list, e.g.
# heston_pass1_kernel<double, (int)8, (int)3, (bool)0, (bool)0> -> heston_pass1_kernelIdLi8ELi3ELb0ELb0E
m = re.search(r"(\w+_kernel)<([^>]*)>", kname)
want = kern
if m:
    parts = []
    for a in m.group(2).split(","):
        a = a.strip()
        if a in ("double", "float"):
            parts.append(a[0])
        else:
            mm = re.match(r"\((int|bool)\)(-?\d+)", a)
            if mm:
                parts.append(("Li" if mm.group(1) == "int" else "Lb") + mm.group(2) + "E")
    want = m.group(1) + "I" + "".join(parts) + "E"
lines = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
    cur_fn, cur_line = None, None
    for l in dis.splitlines():
        if l.startswith(".text.") and l.rstrip().endswith(":"):
            cur_fn = l
            continue
        if cur_fn is None or want not in cur_fn:
            continue
        mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if mm:
            cur_line = (os.path.basename(mm.group(1)), int(mm.group(2)))
            continue
        ma = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if ma and cur_line:
            lines[int(ma.group(1), 16)] = cur_line
samp = collections.Counter(); inst = collections.Counter()
for addr, s, n, src in rows:
    key = lines.get(addr - base, ("?", 0))
    samp[key] += s
    inst[key] += n
tot = sum(samp.values()); itot = sum(inst.values())
srcs = {}
def src_line(f, ln):
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1901_04200_b200", "csrc", f)
    if f not in srcs:
        srcs[f] = open(p).read().splitlines() if os.path.exists(p) else []
    return srcs[f][ln - 1].strip()[:70] if 0 < ln <= len(srcs[f]) else ""
print(f"{kname}\n  samples {tot}, warp-instructions {itot:.3e}")
for key, s in samp.most_common(top):
    print(f"{100*s/tot:5.1f}% stall  {100*inst[key]/itot:5.1f}% inst  {key[0]}:{key[1]:<4d} {src_line(*key)}")
