"""Top SASS lines by sampled warp stalls for one launch of an ncu --set full
capture (source page, SASS view). usage: python tools/stall_lines.py rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
i = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
stall_cols = [(k, h[6:]) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
src = hdr.index("Source")
recs = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    per = {}
    for k, h in stall_cols:
        try:
            per[h] = float(r[k] or 0)
        except ValueError:
            pass
    tot = sum(per.values())
    if tot > 0:
        recs.append((tot, r[0], r[src], sorted(per.items(), key=lambda x: -x[1])[:2]))
grand = sum(x[0] for x in recs) or 1
recs.sort(key=lambda x: -x[0])
for tot, addr, s, why in recs[:top]:
    print(f"{tot / grand:6.1%} {addr} {s[:70]:70s} {', '.join(f'{k} {v:.0f}' for k, v in why)}")
