"""Write profiles/ncu_traffic.json: per-launch DRAM bytes (read + write) of our
kernels from `ncu --set full` reports.  Usage: python tools/ncu_traffic.py rep1 [rep2 ...]"""
import csv, io, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
d = json.load(open(out_path)) if os.path.exists(out_path) else {}
units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, unit_row = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        key = re.search(r"(\w+)\s*[<(]", name.replace("<unnamed>", "")).group(1)
        def val(metric):
            i = hdr.index(metric)
            return float(r[i].replace(",", "")) * units.get(unit_row[i], 1)
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        d[key] = {"dram_bytes_per_launch": b, "read": val("dram__bytes_read.sum"),
                  "write": val("dram__bytes_write.sum"), "kernel": name[:160],
                  "duration_us_under_ncu": val("gpu__time_duration.sum") / 1e3 if unit_row[hdr.index("gpu__time_duration.sum")] == "nsecond" else val("gpu__time_duration.sum"),
                  "report": os.path.basename(rep)}
json.dump(d, open(out_path, "w"), indent=1)
print(json.dumps(d, indent=1))
