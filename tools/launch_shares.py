"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals and shares."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r"(k_[a-zA-Z0-9_]+)", r[ki])
    nm = m.group(1) if m else r[ki][:40]
    tot[nm] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[nm] += 1
T = sum(tot.values())
print(f"total {T/1e3:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{k:28s} {v/1e3:10.3f} ms  {100*v/T:6.2f}%  n={cnt[k]}")
