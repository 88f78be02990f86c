"""Summarise an ncu --set full capture: headline metrics, stall reasons, opcode mix."""
import collections, csv, re, subprocess, sys

rep = sys.argv[1]
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "lts__t_bytes.sum"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]} {units[i]}")
items = [(h, float(v)) for h, v in zip(hdr, vals) if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and v.replace(".", "", 1).isdigit()]
tot = sum(v for _, v in items) or 1
print("-- stall reasons (pc sampling)")
for h, v in sorted(items, key=lambda x: -x[1])[:10]:
    print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * v / tot:5.1f}%")
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout.splitlines()))
h2 = src[1]
i_src, i_s, i_ex = h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)"), h2.index("Instructions Executed")
by, exc = collections.Counter(), collections.Counter()
for r in src[2:]:
    try:
        s, e = int(r[i_s]), int(r[i_ex] or 0)
    except (ValueError, IndexError):
        continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[i_src].strip())
    op = m.group(2).split(".")[0] if m else "?"
    by[op] += s
    exc[op] += e
t2 = sum(by.values()) or 1
print("-- opcode mix (stall samples, executed)")
for op, s in by.most_common(14):
    print(f"  {op:12s} {100 * s / t2:5.1f}%  {exc[op]:>12d}")
