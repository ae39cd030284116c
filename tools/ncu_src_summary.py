"""Summarise an ncu --page source --csv --print-source sass export: stall
samples per opcode and per reason, and the top SASS lines with their reasons.
Usage: python tools/ncu_src_summary.py export.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr, data = rows[1], rows[2:]
i_src, i_all = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
f = lambda r, i: float(r[i] or 0)  # noqa: E731
tot = sum(f(r, i_all) for r in data)
print(f"samples {tot:.0f}")
per_reason = {h: sum(f(r, idx[h]) for r in data) for h in reasons}
print("by reason:", ", ".join(f"{h[6:]} {v / tot * 100:.1f}%" for h, v in sorted(per_reason.items(), key=lambda x: -x[1]) if v))
ops = {}
for r in data:
    t = r[i_src].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] = ops.get(op, 0) + f(r, i_all)
print("by opcode:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
for j, r in sorted(enumerate(data), key=lambda x: -f(x[1], i_all))[:top_n]:
    rs = sorted(((h[6:], f(r, idx[h])) for h in reasons), key=lambda x: -x[1])[:3]
    print(f"{j:4d} {f(r, i_all) / tot * 100:5.2f}%  {r[i_src][:60]:60s} " + " ".join(f"{a}:{b:.0f}" for a, b in rs if b))
