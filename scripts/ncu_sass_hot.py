"""Per-SASS-line instruction counts and stall samples of one kernel in an .ncu-rep (--page source)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
r = list(csv.reader(lines[1:]))
h = r[0]
ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)")
rows = []
for row in r[1:]:
    try:
        rows.append((int(row[ie]), int(row[ss]), row[0], row[1]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in rows); tots = sum(x[1] for x in rows)
print("total instr", tot, "samples", tots)
mode = sys.argv[4] if len(sys.argv) > 4 else "seq"
if mode == "seq":
    for x in rows:
        if x[0] > tot * 0.002 or x[1] > tots * 0.005:
            print(f"{x[0]:>10} {100*x[1]/max(tots,1):5.1f}% {x[2][-5:]} {x[3][:100]}")
else:
    for x in sorted(rows, key=lambda x: -x[1])[:n]:
        print(f"{x[0]:>10} {100*x[1]/max(tots,1):5.1f}% {x[2][-5:]} {x[3][:100]}")
