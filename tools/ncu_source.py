"""Per-CUDA-line instruction and stall totals of one kernel in an ncu report.

    python tools/ncu_source.py report.ncu-rep <function-substring> [top]
"""
import csv
import io
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows, path, func, head = [], None, None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1]
        continue
    if rec[0] == "Function Name":
        func = rec[1]
        continue
    if rec[0] == "Line No":
        head = rec
        continue
    if head and func and kname in func and len(rec) >= 8 and rec[2] == "-":
        rows.append((path.split("/")[-1], rec[0], rec[1], rec[7], rec[4]))


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


tot_i = sum(f(r[3]) for r in rows)
tot_s = sum(f(r[4]) for r in rows)
print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
rows.sort(key=lambda r: -f(r[3]))
for fn, ln, src, i, s in rows[:top]:
    print(f"{fn[:14]:>14}:{ln:<4} {100 * f(i) / max(tot_i, 1):5.1f}% inst {100 * f(s) / max(tot_s, 1):5.1f}% stall | {src.strip()[:90]}")
