"""Top CUDA source lines by warp-level instructions executed from an ncu report (captured with
-lineinfo and --import-source on). Usage: python scripts/ncu_exec_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"], capture_output=True,
                     text=True).stdout
cur, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Name":
        cur = r[1].split("/")[-1]
    elif len(r) >= 3 and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        try:
            e = int(r[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((e, cur, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
print("warp instructions executed", tot)
for e, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * e / tot:5.1f}% {e:9d} {f}:{ln}  {src}")
