"""Summarise an ncu report (raw metrics + per-barrier-segment stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
d = dict(zip(rows[0], rows[2]))
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = []
for h, v in d.items():
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v), h[34:-23]))
        except ValueError:
            pass
st.sort(reverse=True)
print("stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
ist = hdr.index("Warp Stall Sampling (All Samples)")
isrc = hdr.index("Source")
iex = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ist]), r[isrc].strip(), int(r[iex] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in data) or 1
start, acc, inst = 0, 0, 0
for i, (s, srcl, ex) in enumerate(data):
    acc += s
    inst += ex
    if srcl.startswith("BAR") or srcl.startswith("EXIT") or i == len(data) - 1:
        kinds = {}
        for s2, src2, _ in data[start:i + 1]:
            op = src2.split()[0] if src2 else "?"
            if op.startswith("@") and len(src2.split()) > 1:
                op = src2.split()[1]
            op = op.split(".")[0]
            kinds[op] = kinds.get(op, 0) + s2
        top = sorted(kinds.items(), key=lambda x: -x[1])[:6]
        print(f"[{start:5d}-{i:5d}] {100 * acc / tot:5.1f}% samples, {inst:11d} inst, top {top}")
        start, acc, inst = i + 1, 0, 0
