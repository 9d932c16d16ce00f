"""Warp-stall samples of an ncu SASS source export (`--page source --csv --print-source sass`),
printed as a running profile: consecutive instruction windows with their sample share, top
stall reasons and instruction mix, so hot regions (routing phases, fc1/fc2 loops) stand out.
usage: python tools/ncu_sass_regions.py export.csv [window]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 64
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex = float(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    st = {h: float(r[ix[h]] or 0) for h in stall_cols}
    data.append((r[ix["Address"]], r[ix["Source"]].strip(), s, ex, st))
tot = sum(d[2] for d in data)
print(f"instructions {len(data)}, samples {tot:.0f}")
for i in range(0, len(data), win):
    chunk = data[i:i + win]
    s = sum(d[2] for d in chunk)
    if s < 0.005 * tot:
        continue
    st = Counter()
    for d in chunk:
        st.update(d[4])
    ops = Counter(d[1].split()[0] if not d[1].startswith("@") else d[1].split()[1] for d in chunk if d[1])
    ops = Counter({k.split(".")[0]: 0 for k in ops}) + Counter([(d[1].split()[1] if d[1].startswith("@") else d[1].split()[0]).split(".")[0] for d in chunk if d[1]])
    ex = sum(d[3] for d in chunk)
    top = ", ".join(f"{k[6:]}:{100*v/s:.0f}%" for k, v in st.most_common(4))
    print(f"[{i:5d}] {100*s/tot:5.1f}%  exec {ex:9.0f}  {top}  | {', '.join(f'{k}:{v}' for k, v in ops.most_common(6))}")
