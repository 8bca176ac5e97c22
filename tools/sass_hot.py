"""Hot SASS instructions of one kernel in an ncu report (stall samples and
executed counts), to find where a latency-bound kernel spends its time.
  python tools/sass_hot.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
a, s, st, ex = (hdr.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                         "Instructions Executed"))
body = []
for r in rows[2:]:
    if r and r[0] in ("Kernel Name", "Address"):
        if body:
            break  # first matching kernel only
        continue
    if len(r) == len(hdr):
        body.append(r)
tot = sum(float(r[st] or 0) for r in body)
print(f"{len(body)} SASS instructions, {tot:.0f} stall samples, "
      f"{sum(float(r[ex] or 0) for r in body):.0f} warp-instructions executed")
for i, r in sorted(enumerate(body), key=lambda x: -float(x[1][st] or 0))[:top]:
    print(f"{i:5d} {r[a]:>6} {float(r[st] or 0) / max(tot, 1):6.1%} ex={r[ex]:>8}  {r[s][:90]}")
if len(sys.argv) > 5:  # optional: print a range of instruction indices
    lo, hi = int(sys.argv[4]), int(sys.argv[5])
    for i in range(lo, min(hi, len(body))):
        r = body[i]
        print(f"{i:5d} {float(r[st] or 0):5.0f} ex={r[ex]:>6}  {r[s][:100]}")
if len(sys.argv) == 5 and sys.argv[4] == "buckets":
    B = 50
    for b0 in range(0, len(body), B):
        seg = body[b0:b0 + B]
        smp = sum(float(r[st] or 0) for r in seg)
        exe = sum(float(r[ex] or 0) for r in seg)
        if smp or exe:
            print(f"[{b0:5d},{b0 + B:5d}) samples {smp:5.0f} ({smp / max(tot, 1):5.1%}) exec {exe:7.0f}  "
                  f"{seg[0][s][:60]}")
