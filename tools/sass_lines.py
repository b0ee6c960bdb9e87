"""Attribute ncu SASS stall samples to source lines using the local cubin's line table.
python tools/sass_lines.py <sass.csv.gz> <cubin> <kernel-substring> [top]"""
import csv, gzip, io, re, subprocess, sys, collections
path, cubin, kname = sys.argv[1:4]; top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
start = [i for i, l in enumerate(dis) if kname in l and ".text." in l][0]
cur = None; lm = {}
for l in dis[start + 1:]:
    if l.startswith("//----") and ".text." in l: break
    mm = re.search(r'## File "([^"]+)", line (\d+)', l)
    if mm: cur = f'{mm.group(1).split("/")[-1]}:{mm.group(2)}'
    a = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if a and cur: lm[int(a.group(1), 16)] = cur
with gzip.open(path, "rt") as fh:
    lines = fh.read().splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr, body = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
base = int(body[0][ix["Address"]], 16)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
per = collections.defaultdict(lambda: [0, collections.Counter(), 0]); tot = 0
for r in body:
    try: s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError: continue
    off = int(r[ix["Address"]], 16) - base
    key = lm.get(off, "?")
    per[key][0] += s; tot += s
    per[key][2] += int(r[ix["Instructions Executed"]] or 0)
    for c in stall_cols:
        v = int(r[ix[c]] or 0)
        if v: per[key][1][c[6:]] += v
print(f"total samples {tot}")
for k, (s, st, ex) in sorted(per.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*s/tot:5.2f}% {k:28s} ex={ex:<10d} {st.most_common(3)}")
