"""Per-SASS-instruction issue counts and stall samples of one kernel in an ncu report.
usage: python tools/ncu_sass.py <report.ncu-rep> [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ci = {x: i for i, x in enumerate(h)}
st = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
data = rows[hi + 1:]
tot = sum(float(r[ci["# Samples"]] or 0) for r in data)
print("total samples", tot, "instructions executed", sum(float(r[ci["Instructions Executed"]] or 0) for r in data))
for idx, r in enumerate(data):
    s = float(r[ci["# Samples"]] or 0)
    if s / tot < 0.004:
        continue
    tp = sorted(((x, float(r[ci[x]] or 0)) for x in st), key=lambda t: -t[1])[:2]
    print(f"{idx:5d} {100 * s / tot:5.1f}% ie={r[ci['Instructions Executed']]:>8} {r[ci['Source']].strip()[:60]:60s} "
          + " ".join(f"{k[6:]}={100 * x / max(s, 1):.0f}%" for k, x in tp))
