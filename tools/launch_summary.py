"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, mean/total device time and share of the total."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
i_k, i_m, i_v = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
i_u = hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= i_v or r[i_m] != "gpu__time_duration.sum":
        continue
    v = float(r[i_v].replace(",", ""))
    v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[i_u], 1.0)
    name = r[i_k].split("(")[0][:90]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':90s} {'launches':>8s} {'mean_us':>10s} {'total_us':>10s} {'share':>6s}")
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{k:90s} {cnt[k]:8d} {tot[k] / cnt[k]:10.2f} {tot[k]:10.1f} {100 * tot[k] / T:5.1f}%")
