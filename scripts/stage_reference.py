"""Stage the UNMODIFIED reference package into baseline/_ref (git-ignored; travels to the GPU
box with gpurun) for bench.py's reference arm, then apply the test-pinned "variant B" fix.

    python scripts/stage_reference.py

1. copy /root/reference/pkg to a temp dir (the install may write build files into the source
   tree; /root/reference is read-only) and run the offline install the task prescribes:
   pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps
               --target baseline/_ref <copy>
   (--no-deps: its only runtime dependency, numpy, is already in the image; matplotlib,
   needed only by seqplace.plots, is absent and unused here)
2. patch baseline/_ref/seqplace/trajopt.py: as shipped, trajopt._evaluate lacks the
   place_mode parameter that solve_al passes and reads undefined names, so
   every manipulation pipeline raises. The reference's own tests pin "variant B":
       def _evaluate(..., want_grad)  ->  def _evaluate(..., want_grad, place_mode=None)
       + pmode = mode; pquad = pmode == QUADRATIC   (after `quad = mode == QUADRATIC`)
   Nothing else is touched; bench.py then drives the stock seqplace.bench.solve_scene.
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DST = os.path.join(ROOT, "baseline", "_ref")


def apply_variant_b(trajopt_path: str) -> None:
    src = open(trajopt_path).read()
    old_sig = "def _evaluate(values, geo: _Geometry, config: TrajOptConfig, mode, lam, mu, want_grad):"
    if "pmode = mode\n" in src:
        return
    assert src.count(old_sig) == 1, "unexpected reference trajopt.py (signature)"
    src = src.replace(old_sig, old_sig[:-2] + ", place_mode=None):")
    anchor = "    quad = mode == QUADRATIC\n"
    assert src.count(anchor) == 1, "unexpected reference trajopt.py (anchor)"
    src = src.replace(anchor, anchor + "    pmode = mode\n    pquad = pmode == QUADRATIC\n")
    with open(trajopt_path, "w") as f:
        f.write(src)


def main():
    if not os.path.isdir(SRC):
        sys.exit(f"{SRC} not found (run this in the build container)")
    tmp = tempfile.mkdtemp(prefix="spasm_refsrc_")
    shutil.copytree(SRC, os.path.join(tmp, "pkg"))
    shutil.rmtree(DST, ignore_errors=True)
    cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--find-links",
           "/opt/wheelhouse", "--no-deps", "--target", DST, os.path.join(tmp, "pkg")]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        sys.exit(out.stdout + out.stderr)
    apply_variant_b(os.path.join(DST, "seqplace", "trajopt.py"))
    shutil.rmtree(tmp, ignore_errors=True)
    with open(os.path.join(DST, "STAGED.json"), "w") as f:
        json.dump({"source": SRC, "install": " ".join(cmd[2:]), "patch": "variant B (scripts/stage_reference.py)"},
                  f, indent=1)
    print("staged", DST)


if __name__ == "__main__":
    main()
