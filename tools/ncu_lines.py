"""Top source lines (and SASS) by warp-stall samples for one kernel of an ncu report."""
import csv, io, subprocess, sys

path, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
col = 7 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 4  # 4: stall samples, 7: instructions executed
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", kernel, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, tot = [], 0
for r in rows[3:]:
    if len(r) > 4 and r[0]:
        try:
            s = int(r[col])
        except ValueError:
            continue
        lines.append((s, r[0], r[1][:110]))
        tot += s
lines.sort(reverse=True)
print("total samples", tot)
for s, l, src in lines[:top]:
    print(f"{s:7d} {100 * s / max(tot, 1):5.1f}% L{l}: {src}")
