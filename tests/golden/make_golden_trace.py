"""Golden fixtures for the trace / selection-efficacy path (reference bench.py:518-630),
from the REFERENCE itself (stage 1 only; unmodified package):

  * trace_solve on tetris5 and tower4 (scene settings, seed 3): particle ids, selected flags,
    per-step costs and satisfied flags, and the bytes of its export_trace CSV;
  * selection_efficacy on tetris5 (n=1024, m=128, 3 trials) and domino2 (n=256, m=32).

    python tests/golden/make_golden_trace.py   ->  tests/golden/trace.npz
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from seqplace import bench
    from seqplace.problems import load_scene

    out = {}
    for name in ("tetris5", "tower4"):
        tr = bench.trace_solve(load_scene(name), seed=3)
        out[f"{name}_ids"] = tr.particle_ids
        out[f"{name}_selected"] = tr.selected
        out[f"{name}_costs"] = tr.costs
        out[f"{name}_satisfied"] = tr.satisfied
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "t.csv")
            bench.export_trace(tr, p)
            out[f"{name}_csv"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
        print(name, tr.costs.shape, int(tr.selected.sum()), "selected")
    for name, over, trials in (("tetris5", {"n": 1024, "m": 128}, 3), ("domino2", {"n": 256, "m": 32}, 4)):
        s, r = bench.selection_efficacy(load_scene(name), trials=trials, seed=1, solver_overrides=over)
        out[f"eff_{name}"] = np.array([s, r, trials, over["n"], over["m"]], dtype=float)
        print(name, "efficacy", s, r)
    np.savez_compressed(os.path.join(HERE, "trace.npz"), **out)


if __name__ == "__main__":
    main()
