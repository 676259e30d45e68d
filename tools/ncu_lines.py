"""Per-CUDA-source-line instruction counts and stall samples from an .ncu-rep (cuda,sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = None; recs = []; tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            ie = int(r[7] or 0); st = int(r[4] or 0)
        except ValueError:
            continue
        tot += ie
        recs.append((ie, st, fname, r[0], r[1][:100]))
print("total instructions", tot)
for ie, st, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{ie:10d} {100*ie/tot:5.1f}% stall {st:6d}  {f}:{ln}  {src}")
