"""Top CUDA source lines by warp-stall samples from an ncu report (captured with
-lineinfo and --import-source on). Usage: python scripts/ncu_lines.py rep.ncu-rep [N] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    args += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(args, capture_output=True, text=True).stdout
cur, hdr, lines = None, None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif len(r) >= 3 and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        try:
            s = int(r[4] or 0) if r[4] not in ("", "-") else 0
            e = int(r[7] or 0) if r[7] not in ("", "-") else 0
        except ValueError:  # a source line whose text spilled into the numeric columns
            continue
        lines.append((s, e, cur, int(r[0]), r[1].strip()[:100]))
tot = sum(x[0] for x in lines) or 1
byfile = {}
for s, e, f, l, src in lines:
    byfile[f] = byfile.get(f, 0) + s
print("samples", tot, {k: f"{100 * v / tot:.1f}%" for k, v in sorted(byfile.items(), key=lambda x: -x[1])})
for s, e, f, l, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {e:9d} {f}:{l}  {src}")
