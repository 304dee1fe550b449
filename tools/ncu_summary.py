"""One-kernel ncu --set full capture -> a compact JSON summary for profiles/.

    python tools/ncu_summary.py report.ncu-rep cubin kernel_substring src.cu out.json "note" ["regions"]

Metrics from the raw page (duration, instructions, issue, occupancy, pipes,
DRAM bytes, L1/L2 hit rates) and, with regions ("name:lo-hi,..."), the share
of stall samples / instructions and top stalls per source region (ncu_lines.py).
"""
import csv, io, json, subprocess, sys

rep, cubin, kern, srcf, out, note = sys.argv[1:7]
regions = sys.argv[7] if len(sys.argv) > 7 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second"]
metrics = {}
for k in want:
    if k in h:
        v = rows[2][h.index(k)]
        try:
            v = float(v.replace(",", ""))
        except ValueError:
            pass
        metrics[k] = v
res = {"note": note, "source": f"ncu -i {rep} --page raw/source", "metrics": metrics}
if regions:
    txt = subprocess.run([sys.executable, __file__.rsplit("/", 1)[0] + "/ncu_lines.py", rep, cubin, kern, srcf, regions],
                         capture_output=True, text=True).stdout
    reg = {}
    for line in txt.splitlines():
        if line.startswith("region"):
            parts = line.split()
            name = parts[1]
            samp = float(parts[2].rstrip("%"))
            inst = float(parts[4].rstrip("%"))
            stalls = line.split("[", 1)[1].rstrip("]")
            reg[name] = {"stall_samples_pct": samp, "instructions_pct": inst, "top_stalls": stalls}
    res["regions"] = reg
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
