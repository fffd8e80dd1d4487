"""Per-source-line stall samples / instructions from an ncu report (needs -lineinfo)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda"], capture_output=True, text=True).stdout
lines = out.splitlines()
cur = None; rows = []
i = 0
while i < len(lines):
    l = lines[i]
    if l.startswith('"File Name"'):
        cur = next(csv.reader([l]))[1]
        hdr = next(csv.reader([lines[i + 1]]))
        i += 2
        continue
    r = next(csv.reader([l]))
    if cur and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            n = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            s = n = 0
        if s or n:
            rows.append((s, n, cur.split("/")[-1], d["Line No"], d["Source"].strip()[:90]))
    i += 1
tot = sum(r[0] for r in rows)
print("total samples", tot)
for s, n, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {n:11d} {f}:{ln:5s} {src}")
