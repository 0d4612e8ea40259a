"""Per-source-line warp-stall breakdown of one kernel in an ncu report.
usage: python tools/ncu_lines.py <report.ncu-rep> <object.o> <mangled-kernel-substring> [top]"""
import csv, os, re, subprocess, sys, tempfile

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 22
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ci = {x: i for i, x in enumerate(h)}
st = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
data = rows[hi + 1:]
tot = sum(float(r[ci["# Samples"]] or 0) for r in data)
agg = {}
for r in data:
    for x in st:
        agg[x] = agg.get(x, 0) + float(r[ci[x]] or 0)
print(sorted([(k, round(100 * v / tot, 1)) for k, v in agg.items()], key=lambda t: -t[1])[:10])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
offmap, cur, infn = {}, None, False
for l in sass.split("\n"):
    if l.startswith(".text."):
        infn = kname in l
        continue
    if not infn:
        continue
    m2 = re.search(r"line (\d+)", l)
    if "//## File" in l and m2:
        cur = (l.split('"')[1].split("/")[-1] if '"' in l else "?", int(m2.group(1)))
    m3 = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m3:
        offmap[int(m3.group(1), 16)] = cur
base = int(data[0][0], 16)
agg2 = {}
for r in data:
    ln = offmap.get(int(r[0], 16) - base)
    s = float(r[ci["# Samples"]] or 0)
    d = agg2.setdefault(ln, [0, {}])
    d[0] += s
    for x in st:
        d[1][x] = d[1].get(x, 0) + float(r[ci[x]] or 0)
for ln, (v, rs) in sorted(agg2.items(), key=lambda t: -t[1][0])[:top]:
    tp = sorted(rs.items(), key=lambda t: -t[1])[:2]
    print(f"{100 * v / tot:5.1f}% {ln} " + " ".join(f"{k[6:]}={100 * x / max(v, 1):.0f}%" for k, x in tp))
