"""Per-source-line warp-stall samples from an ncu report's `--page source --csv --print-source cuda,sass`
export. usage: python tools/ncu_lines.py export.csv [top_n] [file_filter]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
cur_file, hdr, lines = None, None, []
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    si = 4
    try:
        samp = float(r[si] or 0)
    except ValueError:
        continue
    # stall-reason columns (the 'stall_*' style headers), all samples
    reasons = {}
    for j, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and j < len(r):
            try:
                v = float(r[j] or 0)
            except ValueError:
                continue
            if v:
                reasons[h.replace("Warp Stall Sampling (All Samples)", "").strip()] = v
    lines.append((samp, cur_file, r[0], r[1].strip()[:90], reasons))
tot = sum(x[0] for x in lines)
print(f"total samples {tot:.0f}")
for samp, f, ln, src, rs in sorted([x for x in lines if filt in x[1]], key=lambda x: -x[0])[:top]:
    rr = ", ".join(f"{k}:{v:.0f}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
    print(f"{samp:7.0f} {100*samp/tot:5.1f}% {f}:{ln:5} {src}  [{rr}]")
