"""Map ncu per-instruction stall samples to source lines (needs the cubin with -lineinfo).
usage: python tools/ncu_hot.py <report.ncu-rep> <object.o> <kernel-substring>"""
import csv, re, subprocess, sys, os, tempfile
rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout.split("\n")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
d = {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}
for k in ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread"]:
    print(k, d.get(k))
st = [(h, float(v[0])) for h, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and v[0].replace('.', '', 1).isdigit()]
st.sort(key=lambda t: -t[1]); tot = sum(v for _, v in st)
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100*v/tot:.1f}%" for h, v in st[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(srows) if r and r[0] == "Address")
ci = {h: i for i, h in enumerate(srows[hi])}
data = srows[hi + 1:]
base = int(data[0][0], 16)
offmap, cur, infn = {}, None, False
for l in sass:
    if l.startswith(".text."):
        infn = kname in l
        continue
    if not infn:
        continue
    m2 = re.search(r'line (\d+)', l)
    if "//## File" in l and m2:
        cur = (l.split('"')[1].split('/')[-1] if '"' in l else '?', int(m2.group(1)))
    m3 = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m3:
        offmap[int(m3.group(1), 16)] = cur
agg = {}
tot = sum(float(r[ci['# Samples']] or 0) for r in data)
for r in data:
    ln = offmap.get(int(r[0], 16) - base)
    agg[ln] = agg.get(ln, 0.0) + float(r[ci['# Samples']] or 0)
for ln, v in sorted(agg.items(), key=lambda t: -t[1])[:18]:
    text = ""
    if ln and ln[0] != "?":
        p = os.path.join(os.path.dirname(obj), "..", ln[0]) if False else None
    print(f"{100*v/tot:5.1f}%  {ln}")
