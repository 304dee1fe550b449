"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) for the
last simulation step in it: per kernel launches, time, share, DRAM bytes.
Usage: python tools/launch_summary.py launches.csv out.json "<note>" """
import collections, csv, json, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
I = {h: i for i, h in enumerate(hdr)}
launches = collections.OrderedDict()
for r in rows[1:]:
    if not r[I["ID"]].isdigit():
        continue
    d = launches.setdefault(int(r[I["ID"]]), {"name": r[I["Kernel Name"]]})
    d[r[I["Metric Name"]]] = float(r[I["Metric Value"]].replace(",", ""))
L = list(launches.values())
start = max(i for i, l in enumerate(L) if "kick_drift" in l["name"])  # the last step
step = L[start:]
tot = sum(l["gpu__time_duration.sum"] for l in step)
agg = collections.OrderedDict()
for l in step:
    name = l["name"].split("(")[0]
    a = agg.setdefault(name, {"launches": 0, "ns_total": 0.0, "dram_bytes": 0.0})
    a["launches"] += 1
    a["ns_total"] += l["gpu__time_duration.sum"]
    a["dram_bytes"] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
for a in agg.values():
    a["share_of_step_kernels"] = a["ns_total"] / tot
out = {"_note": sys.argv[3] if len(sys.argv) > 3 else "",
       "step_kernel_ns": tot, "launches_in_step": len(step),
       "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["ns_total"]))}
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, a in list(out["kernels"].items())[:12]:
    print(f"{a['ns_total']/1e3:9.1f} us {100*a['share_of_step_kernels']:5.1f}%  x{a['launches']:2d} {a['dram_bytes']/1e6:8.1f} MB  {k[:70]}")
