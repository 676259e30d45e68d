"""Instructions / stall samples per source-line range of one file in an .ncu-rep."""
import csv, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = [tuple(int(v) for v in r.split("-")) for r in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; acc = {r: [0, 0] for r in ranges}; tot = [0, 0]
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            ln, ie, st = int(r[0]), int(r[7] or 0), int(r[4] or 0)
        except ValueError:
            continue
        tot[0] += ie; tot[1] += st
        if cur == fname:
            for a, b in ranges:
                if a <= ln <= b:
                    acc[(a, b)][0] += ie; acc[(a, b)][1] += st
print("total inst %d stalls %d" % tuple(tot))
for k, (ie, st) in acc.items():
    print("%5d-%-5d inst %10d (%5.1f%%)  stall %6d (%5.1f%%)" % (k[0], k[1], ie, 100 * ie / tot[0], st, 100 * st / max(tot[1], 1)))
