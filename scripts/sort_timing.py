"""Device time of spasm_sort_pairs (stable key/index sort) per n, fp32 keys with ties
(diagnostic; CUDA events on the launching stream, median of 50 sorts after warm-up).
Usage: python scripts/sort_timing.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2510_07674_b200 import _native as nat  # noqa: E402

lib = nat.load()
s = nat.stream_handle()
for n in (1024, 2048, 4096, 8192, 16384, 65536):
    rng = np.random.default_rng(n)
    c = torch.as_tensor(np.floor(rng.uniform(0, 5000, size=n)) * 0.125, device="cuda", dtype=torch.float32)
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    vals = torch.empty(n, dtype=torch.int32, device="cuda")
    nb = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.empty(max(1, lib.spasm_sort_workspace_bytes(nat.F32, n)), dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(60):
        nat.check(lib.spasm_cost_keys(nat.F32, nat.ptr(c), n, float("inf"), nat.ptr(keys), nat.ptr(vals), nat.ptr(nb),
                                      s), "keys")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nat.check(lib.spasm_sort_pairs(nat.F32, nat.ptr(keys), nat.ptr(vals), n, nat.ptr(ws), s), "sort")
        e1.record()
        torch.cuda.synchronize()
        if it >= 10:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"n={n:6d}: sort {np.median(ts):7.1f} us")
