"""cProfile of the host side of solve_scene (C2 tower3c by default): where the time between
kernels goes. Usage: python scripts/host_profile.py [scene] [solves]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2510_07674_b200.bench_api import solve_scene  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tower3c"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
scene = load_scene(name)
model = as_cost_model(scene.problem, precision="fp32")
for s in range(3):
    solve_scene(scene, seed=100 + s, model=model)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(n):
    solve_scene(scene, seed=s, model=model)
torch.cuda.synchronize()
print(f"plain: {(time.perf_counter() - t0) / n * 1e3:.3f} ms per solve")
pr = cProfile.Profile()
pr.enable()
for s in range(n):
    solve_scene(scene, seed=s, model=model)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
