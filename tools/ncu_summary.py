"""Summarise an ncu report: key counters, stall reasons, hottest source lines."""
import csv, subprocess, sys, io

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def raw():
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


hdr, kernels = raw()
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second"]
for k in kernels:
    for key in keys:
        if key in hdr:
            print(f"{key:70s} {k[hdr.index(key)]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(k[i])
            except ValueError:
                continue
            if v > 0.05:
                st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    print("stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)))

if top:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, fname = [], None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0].isdigit() and len(r) > 8 and r[2] == "-":
            n = int(r[7] or 0)
            if n:
                agg.append((n, int(r[8] or 0) / n, int(r[4] or 0), fname, r[0], r[1][:90]))
    tot = sum(a[0] for a in agg) or 1
    stot = sum(a[2] for a in agg) or 1
    agg.sort(reverse=True)
    print(f"total warp instructions {tot}")
    for n, th, smp, f, ln, src in agg[:top]:
        print(f"{100*n/tot:5.2f}% thr{th:5.1f} stall{100*smp/stot:5.1f}% {f}:{ln:>4s} {src}")
