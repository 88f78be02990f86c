"""Stall samples aggregated by CUDA source line (needs -lineinfo + --import-source)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
# find header row containing 'Source'
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_line = hdr.index("Line") if "Line" in hdr else None
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[i_s]), r[i_line] if i_line is not None else "", r[i_src]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for s, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  L{ln:>5s}  {src.strip()[:100]}")
