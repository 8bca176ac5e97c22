"""Stall samples per CUDA source line of one kernel in an ncu report.
  python tools/src_hot.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, cur, stats, seen_fn = "?", None, {}, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        seen_fn += 1
        if seen_fn > 50:
            break
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ei = hdr.index("Instructions Executed")
        continue
    if r[0]:  # a source line row
        cur = (fname, int(r[0]), r[1].strip()[:80])
        st = stats.setdefault(cur, [0.0, 0.0])
        try:
            st[0] += float(r[si] or 0)
            st[1] += float(r[ei] or 0)
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in stats.values()) or 1
for (f, ln, src), (smp, ex) in sorted(stats.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{smp / tot:6.1%} ex={ex:>10.0f} {f}:{ln:<5d} {src}")
