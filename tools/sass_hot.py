"""Hot-spot view of an ncu `--page source --csv --print-source sass` export (gzip ok).
python tools/sass_hot.py file.sass.csv.gz [top]  -> top instructions by stall samples, plus
per-opcode totals (samples, executed warp instructions)."""
import csv, gzip, io, sys, collections
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as fh:
    lines = fh.read().splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr, body = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0; ops = collections.defaultdict(lambda: [0, 0]); recs = []
for r in body:
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0); ex = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[ix["Source"]].strip(); opc = src.split()[0] if src else "?"
    if opc.startswith("@"): opc = src.split()[1]
    opc = opc.split(".")[0]
    ops[opc][0] += s; ops[opc][1] += ex; tot += s
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    recs.append((s, r[ix["Address"]][-5:], src[:70], ex, st))
print(f"total samples {tot}")
print("by opcode (samples%, warp-insts):")
for k, (s, e) in sorted(ops.items(), key=lambda x: -x[1][0])[:25]:
    print(f"  {k:10s} {100*s/tot:5.1f}%  {e}")
print("top instructions:")
for s, a, src, ex, st in sorted(recs, key=lambda x: -x[0])[:top]:
    print(f"  {100*s/tot:5.2f}% {a} {src:70s} ex={ex} {st}")
