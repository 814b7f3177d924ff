"""Aggregate ncu per-SASS-instruction stall samples (source page) by opcode and
list the hottest instructions.  python tools/sass_stalls.py report.ncu-rep [top]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = collections.Counter()
by_reason = collections.Counter()
tot = 0
recs = []
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += n
    by_op[op.split(".")[0]] += n
    for h in stall_cols:
        v = r[ix[h]]
        if v and v != "0":
            by_reason[h] += int(v)
    recs.append((n, r[ix["Address"]], src, {h: r[ix[h]] for h in stall_cols if r[ix[h]] not in ("", "0")}))
print(f"total samples {tot}")
print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in by_reason.most_common(12)))
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in by_op.most_common(15)))
for n, a, src, st in sorted(recs, reverse=True)[:top]:
    print(f"{n:7d} {a[-5:]} {src[:60]:60s} {st}")
