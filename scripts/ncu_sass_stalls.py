"""Per-SASS-instruction stall samples of one kernel in an ncu report (warp sampling with
--import-source on), grouped into address windows. Usage:
python scripts/ncu_sass_stalls.py rep.ncu-rep [window_instructions] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 64
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
hdr, rows = None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0].startswith("0x"):
        rows.append(r)
ix = {k: i for i, k in enumerate(hdr)}


def num(r, k):
    v = r[ix[k]]
    try:
        return float(v)
    except ValueError:
        return 0.0


keys = ["stall_no_inst", "stall_wait", "stall_barrier", "stall_short_sb", "stall_selected", "stall_branch_resolving"]
tot = {k: sum(num(r, k) for r in rows) for k in keys}
S = sum(num(r, "Warp Stall Sampling (All Samples)") for r in rows)
E = sum(num(r, "Instructions Executed") for r in rows)
print(f"{len(rows)} SASS instructions, {S:.0f} samples, {E:.0f} warp instructions executed")
print("  " + ", ".join(f"{k[6:]} {tot[k] / S * 100:.1f}%" for k in keys))
wins = []
for i in range(0, len(rows), win):
    chunk = rows[i:i + win]
    s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in chunk)
    e = sum(num(r, "Instructions Executed") for r in chunk)
    ni = sum(num(r, "stall_no_inst") for r in chunk)
    wt = sum(num(r, "stall_wait") for r in chunk)
    br = sum(num(r, "stall_barrier") for r in chunk)
    ops = {}
    for r in chunk:
        op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    common = ",".join(f"{k}{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:4])
    wins.append((s, i, e, ni, wt, br, common))
print(f"top windows of {win} instructions by samples: start index, samples %, executed, no_inst %, wait %, barrier %, ops")
for s, i, e, ni, wt, br, common in sorted(wins, reverse=True)[:top]:
    print(f"  {i:6d} {s / S * 100:5.1f}% exec {e:9.0f}  no_inst {ni / S * 100:4.1f}%  wait {wt / S * 100:4.1f}%  "
          f"barrier {br / S * 100:4.1f}%  {common}")
