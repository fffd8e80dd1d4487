"""Summarise an ncu source page (SASS): instructions and stall samples per opcode."""
import csv, subprocess, sys, collections, re
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter(); stalls = collections.Counter(); thr = collections.Counter()
top = []
for r in rows[1:]:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
    if not m: continue
    op = m.group(2).split(".")[0]
    if not r[ix["Instructions Executed"]].isdigit(): continue
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    t = int(r[ix["Predicated-On Thread Instructions Executed"]] or 0)
    ops[op] += n; stalls[op] += s; thr[op] += t
    top.append((s, src, n))
tot = sum(ops.values()); stot = sum(stalls.values())
print(f"total warp-instr {tot:.3e}  stall samples {stot}")
for op, n in ops.most_common(40):
    print(f"{op:10s} {n:12.3e} {100*n/tot:5.1f}%  stalls {100*stalls[op]/max(stot,1):5.1f}%  thr/inst {thr[op]/max(n,1):5.1f}")
print("--- top stalled instructions")
for s, src, n in sorted(top, reverse=True)[:25]:
    print(f"{s:6d} {n:10d}  {src}")
