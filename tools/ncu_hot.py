"""Hottest SASS lines of one kernel in an ncu report (warp-stall samples + executed instructions).
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[hi + 1:] if len(r) > ei and r[0].startswith("0x")]
tot = sum(float(r[wi] or 0) for r in body) or 1
print(f"{len(body)} SASS lines, {tot:.0f} stall samples, {sum(float(r[ei] or 0) for r in body):.0f} warp instructions")
for r in sorted(body, key=lambda r: -float(r[wi] or 0))[:top]:
    print(f"{float(r[wi] or 0) / tot:6.1%} {r[ei]:>8s}  {r[0][-5:]} {r[si].strip()[:90]}")
