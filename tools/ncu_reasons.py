"""Warp-stall reason breakdown (pc sampling) of an .ncu-rep."""
import csv, subprocess, sys
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
    pre = "smsp__pcsamp_warps_issue_stalled_"
    items = []
    for k, x in d.items():
        if k.startswith(pre) and not k.endswith("not_issued"):
            try: items.append((k[len(pre):], float(x.replace(",", ""))))
            except ValueError: pass
    tot = sum(v for _, v in items) or 1
    print(rep, "samples", int(tot))
    print("  " + "  ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(items, key=lambda t: -t[1])[:9]))
