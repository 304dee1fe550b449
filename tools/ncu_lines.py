"""Per-source-line stall samples / instructions of one kernel from an ncu report.

    python tools/ncu_lines.py report.ncu-rep cubin kernel_mangled_substring src.cu [regions]

Inlined header code (e.g. the FFMA2 intrinsics) is charged to the last line of
src.cu seen before it in the disassembly.  regions: "name:lo-hi,name:lo-hi"
sums the share of source-line ranges.
"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, cubin, kern, srcf = sys.argv[1:5]
regions = sys.argv[5] if len(sys.argv) > 5 else ""
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
m, cur, inside = {}, None, False
for l in dis:
    if l.startswith(".text.") or l.startswith("//---------------------"):
        if inside and m:
            break
        inside = kern in l
        continue
    if not inside:
        continue
    f = re.search(r'//## File "(.*?)", line (\d+)', l)
    if f and f.group(1).endswith(srcf.split("/")[-1]):
        cur = int(f.group(2))
    a = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if a and cur:
        m[int(a.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iW, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[2:]:  # the first profiled launch only
    if not r or not re.fullmatch(r"[0-9a-fA-Fx]+", r[0]):
        break
    data.append(r)
base = int(data[0][0], 16)
W, I = defaultdict(float), defaultdict(float)
stall_cols = [(i, c.replace("stall_", "")) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
ST = defaultdict(lambda: defaultdict(float))
for r in data:
    ln = m.get(int(r[0], 16) - base, -1)
    W[ln] += float(r[iW] or 0)
    I[ln] += float(r[iI] or 0)
    for i, c in stall_cols:
        ST[ln][c] += float(r[i] or 0)
tw, ti = sum(W.values()), sum(I.values())
src = open(srcf).read().split("\n")
print(f"samples {tw:.0f}  warp-instructions {ti:.4g}")
for ln in sorted(W, key=lambda k: -W[k])[:40]:
    print(f"{ln:5d} {W[ln] / tw * 100:5.1f}% samp {I[ln] / ti * 100:5.1f}% inst | "
          f"{src[ln - 1].strip()[:90] if ln > 0 else ''}")
for reg in filter(None, regions.split(",")):
    name, rng = reg.split(":")
    lo, hi = map(int, rng.split("-"))
    w = sum(v for k, v in W.items() if lo <= k <= hi)
    i = sum(v for k, v in I.items() if lo <= k <= hi)
    st = defaultdict(float)
    for k, d in ST.items():
        if lo <= k <= hi:
            for c, v in d.items():
                st[c] += v
    tops = ", ".join(f"{c} {v / max(w, 1) * 100:.0f}%" for c, v in sorted(st.items(), key=lambda kv: -kv[1])[:6])
    print(f"region {name:12s} {w / tw * 100:5.1f}% samp {i / ti * 100:5.1f}% inst ({i:.3g})  [{tops}]")
