"""Executed-instruction census from one tools/gpu_profile.sh session.

Reads gpurun_out/<TAG>_cfg3{,f32}_z{0,1}_raw.csv.gz (ncu --set full, raw page)
and gpurun_out/<TAG>_census_<cfg>_<prec>_z{0,1}.csv (ncu --csv metric logs) and
prints the EXECUTED / DRAM tables of paper_1901_04200_b200/census.py: thread-
level DADD+DMUL+DFMA (fp32 mode: FADD+FMUL+FFMA) with predicate on per path of
the launch, and DRAM bytes per path. z0 = LTG_ZSTORE=0 (pass 2 regenerates its
draws), z1 = every chunk's draws stored.

usage: census_from_ncu.py TAG [dir]
"""
import csv
import gzip
import io
import os
import sys

TAG = sys.argv[1]
DIR = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
OPS = {"fp64": ("dadd", "dmul", "dfma"), "fp32": ("fadd", "fmul", "ffma")}
PATHS = {"cfg3": 1 << 20, "cfg1": 1 << 16, "cfg2": 1 << 18, "cfg4": 1 << 18}
NAMES = {"cfg3": "cfg3_heston", "cfg1": "cfg1_gbm", "cfg2": "cfg2_localvol", "cfg4": "cfg4_basket16"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        # durations in ns
        "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6,
        "second": 1e9}


def num(s):
    return float(s.replace(",", ""))


def raw_page(path):
    """[(kernel name, {metric: value in base units})] of an ncu raw-page CSV"""
    rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            try:
                d[h] = num(v) * UNIT.get(u, 1.0)
            except ValueError:
                pass
        out.append((r[hdr.index("Kernel Name")], d))
    return out


def metric_log(path):
    """the same from an ncu --csv --log-file metric list (one row per metric)"""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    by_id = {}
    for r in rows[1:]:
        k = (r[ix["ID"]], r[ix["Kernel Name"]])
        by_id.setdefault(k, {})[r[ix["Metric Name"]]] = num(r[ix["Metric Value"]]) * UNIT.get(
            r[ix["Metric Unit"]], 1.0)
    return [(k[1], d) for k, d in by_id.items()]


def per_path(d, prec, paths):
    ex = sum(d[f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum"] for o in OPS[prec]) / paths
    dram = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / paths
    return ex, dram, d["gpu__time_duration.sum"] / 1e6, d.get("smsp__inst_executed.sum", 0.0) / paths


def load(cfg, prec, z):
    tag = f"{TAG}_{cfg}{'f32' if prec == 'fp32' else ''}_z{z}_raw.csv.gz"
    p = os.path.join(DIR, tag)
    if os.path.exists(p):
        return raw_page(p)
    p = os.path.join(DIR, f"{TAG}_census_{cfg}_{prec}_z{z}.csv")
    return metric_log(p) if os.path.exists(p) else None


executed, dram, times = {}, {}, {}
for cfg in ("cfg3", "cfg1", "cfg2", "cfg4"):
    for prec in ("fp64", "fp32"):
        e, dr = {}, {}
        for z in (0, 1):
            ks = load(cfg, prec, z)
            if not ks:
                continue
            for name, d in ks:
                which = "pass1" if "pass1" in name else "pass2" if "pass2" in name else None
                if which is None:
                    continue
                ex, by, ms, wi = per_path(d, prec, PATHS[cfg])
                key = which if which == "pass1" and z == 0 else (
                    "pass1_store" if which == "pass1" else "pass2_regen" if z == 0 else "pass2_store")
                if key != "pass1_store":
                    e[key] = round(ex, 1)
                dr[key] = round(by, 1)
                times[(cfg, prec, key)] = (ms, wi)
        if e:
            executed[(NAMES[cfg], prec)] = e
            dram[(NAMES[cfg], prec)] = dr

print("EXECUTED = {")
for k, v in executed.items():
    print(f"    {k!r}: {v!r},")
print("}\nDRAM = {")
for k, v in dram.items():
    print(f"    {k!r}: {v!r},")
print("}\n# kernel ms (ncu, serialised) and warp instructions per path:")
for k, (ms, wi) in times.items():
    print(f"#   {k[0]} {k[1]} {k[2]:12s} {ms:8.3f} ms  {wi:10.1f} warp-inst/path")
