"""Aggregate an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
ii = hdr.index('ID')
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        v = float(r[vi].replace(',', ''))
    except ValueError:
        continue
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki].split('(')[0][:64]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get('gpu__time_duration.sum', 0.0)
    a[2] += m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':66s} {'n':>5s} {'total_us':>10s} {'share':>6s} {'avg_us':>9s} {'GB/s':>8s} {'MB/launch':>10s}")
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:66s} {c:5d} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {t / c / 1e3:9.1f} {b / t if t else 0:8.0f} {b / c / 1e6:10.1f}")
