"""Per-CUDA-line warp-stall samples (where time goes) from an .ncu-rep."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); fname = None; recs = []; tot = 0; toti = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try: ie = int(r[7] or 0); st = int(r[4] or 0)
        except ValueError: continue
        tot += st; toti += ie; recs.append((st, ie, fname, r[0], r[1][:90]))
print("stall samples", tot, "instructions", toti)
for st, ie, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{st:7d} {100*st/tot:5.1f}%  inst {ie:10d}  {f}:{ln}  {src}")
