"""Summarise an ncu launch list (gpu__time_duration.sum CSV) for our kernels."""
import collections, csv, sys

path, out_path, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    v = float(r[iv].replace(",", "")) * scale[r[iu]]
    short = r[ik].split("(")[0].replace("void ", "")[:70]
    tot[short] += v
    cnt[short] += 1
ours = {k: v for k, v in tot.items() if "syscd::" in k}
T = sum(ours.values()) or 1.0
out = [f"# {title}",
       "# ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised per-launch times.",
       "# Our kernels only (torch launches are data generation / setup outside the timed region).", ""]
for k, v in sorted(ours.items(), key=lambda x: -x[1]):
    out.append(f"{v:12.1f} us total {v / cnt[k]:11.1f} us/launch  x{cnt[k]:3d} {100 * v / T:5.1f}%  {k}")
open(out_path, "w").write("\n".join(out) + "\n")
print("\n".join(out))
