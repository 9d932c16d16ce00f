"""Top SASS lines by warp-stall samples (with the dominant stall reasons) from an
`ncu --page source --csv --print-source sass` dump.

usage: python tools/ncu_hot.py dump.csv [N] [--range START END]   (addresses: last 5 hex digits)
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 30
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
seen, data = set(), []
for r in rows[hdr_i + 1:]:
    if len(r) == len(hdr) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
val = lambda r, i: int(float(r[i] or 0))
tot = sum(val(r, i_s) for r in data)
print("total samples", tot, "instructions", sum(val(r, i_e) for r in data))
agg = {h: sum(val(r, i) for r in data) for i, h in stalls}
print("by reason:", ", ".join(f"{h[6:]}={100.0 * v / max(tot, 1):.1f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
if "--range" in sys.argv:
    a = sys.argv.index("--range")
    lo, hi = int(sys.argv[a + 1], 16), int(sys.argv[a + 2], 16)
    sel = [r for r in data if lo <= int(r[0][-5:], 16) <= hi]
    st = sum(val(r, i_s) for r in sel)
    print(f"range {sys.argv[a+1]}..{sys.argv[a+2]}: {st} samples ({100.0 * st / max(tot, 1):.1f}%)")
    for r in sel:
        top = sorted(((val(r, i), h[6:]) for i, h in stalls), reverse=True)[:2]
        print(f"{val(r, i_s):6d} e={val(r, i_e):7d} {r[0][-5:]} {r[1].strip()[:60]:60s} {top[0][1]}={top[0][0]} {top[1][1]}={top[1][0]}")
    sys.exit(0)
for r in sorted(data, key=lambda r: -val(r, i_s))[:n]:
    top = sorted(((val(r, i), h[6:]) for i, h in stalls), reverse=True)[:2]
    print(f"{val(r, i_s):7d} {100.0 * val(r, i_s) / max(tot, 1):5.1f}%  e={val(r, i_e):8d}  {r[0][-5:]}  {r[1].strip()[:70]:70s} {top[0][1]}={top[0][0]} {top[1][1]}={top[1][0]}")
