"""Group an ncu --csv launch list (gpu__time_duration.sum) by kernel: launches, total,
per-launch time and share.  usage: python tools/ncu_launches.py launches.csv [skip-regex]"""
import collections, csv, re, sys

path = sys.argv[1]
skip = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0] if not r[ki].startswith("void ") else r[ki][5:].split("(")[0]
    if skip and skip.search(name):
        continue
    a = agg[name]
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) / 1e3
tot = sum(v[1] for v in agg.values()) or 1.0
print(f"# {sum(v[0] for v in agg.values())} launches")
print("launches    total_us  per_launch_us  share  kernel")
for name, (n, us) in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"{n:8d}  {us:10.1f}  {us / n:13.1f}  {100 * us / tot:5.1f}%  {name[:70]}")
