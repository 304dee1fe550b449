"""Sort / scan kernels of the last step in an ncu launch-list CSV: time, DRAM bytes, GB/s."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
I = {h: i for i, h in enumerate(rows[0])}
L = collections.OrderedDict()
for r in rows[1:]:
    if not r[I["ID"]].isdigit():
        continue
    d = L.setdefault(int(r[I["ID"]]), {"name": r[I["Kernel Name"]]})
    d[r[I["Metric Name"]]] = float(r[I["Metric Value"]].replace(",", ""))
L = list(L.values())
start = max(i for i, l in enumerate(L) if "k_sort_zero" in l["name"])
tot = 0
for l in L[start:]:
    t = l["gpu__time_duration.sum"] / 1e3
    b = (l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)) / 1e6
    tot += t
    print(f"{l['name'].split('(')[0][-24:]:24s} {t:8.1f} us {b:8.1f} MB {b / max(t, 1e-9):6.2f} TB/s")
print("total", round(tot, 1), "us")
