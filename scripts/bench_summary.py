"""One-line summaries of bench JSON files. Usage: python scripts/bench_summary.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable:", exc)
        continue
    bd = line.get("breakdown") or {}
    ro = line.get("reference_outcomes") or {}
    print(f"{f}: p50 {line['p50_solve_ms']:.3f} ms, value {line['value']:.3g}, success {line['success_rate']}, "
          f"al {bd.get('al_device_ms_mean')}, stage1 {bd.get('stage1_ms_mean')}, frac {line['roofline']['frac']:.4g}, "
          f"ref same {ro.get('same_outcome')}/{ro.get('seeds_compared')}, clk {line['clocks']['sm_mhz']}")
