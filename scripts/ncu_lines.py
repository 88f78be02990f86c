"""Per CUDA source line (rows with a line number in the cuda,sass source view):
instructions executed and stall samples of an ncu --set full --import-source capture."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, fname = [], ""
for r in csv.reader(out):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            rows.append((float(r[7] or 0), float(r[4] or 0), fname, r[0], r[1]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows) or 1
tots = sum(x[1] for x in rows) or 1
print(f"total warp instructions executed {tot:.4g}; stall samples {tots:.4g}")
for v, st, f, ln, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100*v/tot:5.1f}% inst {100*st/tots:5.1f}% samp  {f}:{ln:>4s}  {src.strip()[:80]}")
print("-- by stall samples")
for v, st, f, ln, src in sorted(rows, key=lambda x: -x[1])[:top // 2]:
    print(f"{100*v/tot:5.1f}% inst {100*st/tots:5.1f}% samp  {f}:{ln:>4s}  {src.strip()[:80]}")
