"""Executed-instruction mix of one kernel from an ncu report (SASS source page).
Usage: python tools/sass_mix.py report.ncu-rep [units_per_launch]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Source" in r)
start = rows.index(hdr) + 1
i_src, ix = hdr.index("Source"), hdr.index("Instructions Executed")
i_st = hdr.index("Warp Stall Sampling (All Samples)")
c, st = collections.Counter(), collections.Counter()
tot = 0
for r in rows[start:]:
    if len(r) <= ix:
        continue
    try:
        n = int(r[ix] or 0)
    except ValueError:
        continue
    op = r[i_src].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    c[o] += n
    st[o] += int(r[i_st] or 0)
    tot += n
ts = sum(st.values()) or 1
for o, n in c.most_common(45):
    per = f" per-unit {n * 32 / units:7.2f}" if units else ""
    print(f"{o:10s} {n:12d} {100 * n / tot:5.1f}% stall {100 * st[o] / ts:5.1f}%{per}")
print("total warp instructions", tot, f"per-unit(thread-instr) {tot * 32 / units:.1f}" if units else "")
