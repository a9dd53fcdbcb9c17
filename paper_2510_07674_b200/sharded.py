"""Multi-GPU stage 1: ``particle_opt.solve`` with each restart's particles sharded across
ranks (one process per GPU, ``torch.distributed`` over NCCL). SURVEY.md 8e.

Partitioning follows the reference's own row chunking (``_BatchOps``, reference
particle_opt.py:146-173): rank r owns the contiguous rows ``np.array_split`` would give it,
of the ONE centralized draw of the restart (particle_opt.py:176-192). Per restart:

1. ``spasm_shard_select`` (device): sample + LINEAR-evaluate the rank's rows, stable-sort
   them, emit the rank's elite run (m records ``(order key, global row)``).
2. all-gather of the elite runs (m x 16 B per rank). When that gather is large
   (world x m x 16 B > SELECT_PROTOCOL_BYTES) the exact distributed top-m select replaces
   it (``topm_exchange``): an MSB-first radix select of the global m-th key over
   all-reduced 256-bin digit counts, then each rank contributes only its records of the
   global top m (m records in total instead of world x m).
3. ``spasm_shard_descend`` (device): exact merge of the runs into the global stable top-m
   (particle_opt.py:195-200), re-draw of the rank's slice of it, fused descent schedule
   (particle_opt.py:266-300), satisfying ordering and re-check (particle_opt.py:359-366).
4. all-gather of the per-rank candidate blocks (p_return records), host merge by
   (cost, position) = the reference's stable order over the satisfying rows.

No collective runs inside the step loop. The result (success, particles, costs, indices,
restarts) is identical to the single-GPU ``solve`` for every world size; only
``report.device_ms`` and ``report.launches`` are per rank.
"""
from __future__ import annotations

import time
from typing import Optional

import numpy as np

from . import _native as nat
from .particle_opt import (
    _SAMPLERS,
    NativeCostModel,
    OptimizerConfig,
    SolveReport,
    SolveResult,
    ctypes_byref,
    torch_dtype,
)


def _torch():
    import torch

    return torch


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous chunk, np.array_split(range(n), world) semantics."""
    q, r = divmod(int(n), int(world))
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


class TorchComm:
    """All-gather over a torch.distributed process group (NCCL on device tensors; gloo
    stages through host memory). ``group=None`` with no initialised process group is a
    world of one."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.active = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.active else 0
        self.world = dist.get_world_size(group) if self.active else 1
        self.backend = dist.get_backend(group) if self.active else None

    def all_reduce_sum(self, t):
        """Elementwise sum over the ranks (t's device; gloo stages through host memory)."""
        if self.world == 1:
            return t
        import torch.distributed as dist

        if self.backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            return t
        src = t.detach().cpu().contiguous()
        dist.all_reduce(src, op=dist.ReduceOp.SUM, group=self.group)
        return src.to(t.device)

    def all_gather(self, t):
        """(world, *t.shape) tensor on t's device, rank-major."""
        torch = _torch()
        if self.world == 1:
            return t.unsqueeze(0)
        import torch.distributed as dist

        if self.backend == "nccl":
            out = torch.empty((self.world, *t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        src = t.detach().cpu().contiguous()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        return torch.stack(parts).to(t.device)


class NativeShardOps:
    """Device halves of a sharded restart through the libspasm C-ABI."""

    def __init__(self, model: NativeCostModel, config: OptimizerConfig, sampler: int, warm: Optional[np.ndarray],
                 n_local_max: int, m_local_max: int):
        torch = _torch()
        nat.require_cuda()
        self.model = model
        self.lib = nat.load()
        self.cfg = config.native(sampler)
        self.m = config.m
        self.p = config.p_return
        self.D = model.dimension
        self.warm = None
        self.n_warm = 0
        if warm is not None and len(warm):
            self.warm = torch.as_tensor(np.ascontiguousarray(warm, dtype=float), device="cuda")
            self.n_warm = self.warm.shape[0]
        nbytes = self.lib.spasm_shard_workspace_bytes(model.handle, model.dtype_id, ctypes_byref(self.cfg),
                                                      n_local_max, m_local_max)
        self.ws = torch.empty(max(1, nbytes), dtype=torch.uint8, device="cuda")
        self.launches = 0

    @property
    def key_bits(self) -> int:
        return 32 if self.model.dtype_id == nat.F32 else 64

    def select(self, restart: int, row_lo: int, n_local: int, elite: bool = True):
        """Sample + evaluate + sort the rank's rows; with ``elite`` also emit its elite run
        (all-gather protocol); the top-m select protocol reads the sorted keys in place."""
        torch = _torch()
        self.n_local = n_local
        out = torch.empty((self.m, 2), dtype=torch.int64, device="cuda") if elite else None
        nl = nat.c_int32(0)
        nat.check(self.lib.spasm_shard_select(self.model.handle, self.model.dtype_id, ctypes_byref(self.cfg), restart,
                                              row_lo, n_local, nat.ptr(self.warm), self.n_warm, nat.ptr(self.ws),
                                              self.ws.numel(), nat.ptr(out), ctypes_byref(nl),
                                              nat.stream_handle()), "shard_select")
        self.launches += nl.value
        return out

    def topm_init(self):
        torch = _torch()
        st = torch.empty(int(self.lib.spasm_shard_topm_state_bytes()), dtype=torch.uint8, device="cuda")
        nat.check(self.lib.spasm_shard_topm_init(self.model.dtype_id, self.m, nat.ptr(st), nat.stream_handle()),
                  "shard_topm_init")
        return st

    def topm_hist(self, st):
        torch = _torch()
        h = torch.empty(256, dtype=torch.int64, device="cuda")
        nat.check(self.lib.spasm_shard_topm_hist(self.model.handle, self.model.dtype_id, ctypes_byref(self.cfg),
                                                 self.n_local, nat.ptr(self.ws), nat.ptr(st), nat.ptr(h),
                                                 nat.stream_handle()), "shard_topm_hist")
        self.launches += 1
        return h

    def topm_pick(self, st, hist_sum):
        nat.check(self.lib.spasm_shard_topm_pick(nat.ptr(st), nat.ptr(hist_sum.contiguous()), nat.stream_handle()),
                  "shard_topm_pick")
        self.launches += 1

    def topm_local(self, st):
        torch = _torch()
        c = torch.empty(3, dtype=torch.int64, device="cuda")
        nat.check(self.lib.spasm_shard_topm_local(self.model.handle, self.model.dtype_id, ctypes_byref(self.cfg),
                                                  self.n_local, nat.ptr(self.ws), nat.ptr(st), nat.ptr(c),
                                                  nat.stream_handle()), "shard_topm_local")
        self.launches += 1
        return c

    def topm_contrib(self, take: int, cap: int):
        torch = _torch()
        rec = torch.empty((cap, 2), dtype=torch.int64, device="cuda")
        nat.check(self.lib.spasm_shard_topm_contrib(self.model.handle, self.model.dtype_id, ctypes_byref(self.cfg),
                                                    self.n_local, nat.ptr(self.ws), take, cap, nat.ptr(rec),
                                                    nat.stream_handle()), "shard_topm_contrib")
        self.launches += 1
        return rec

    def descend(self, restart: int, runs, pos_lo: int, pos_hi: int):
        """``runs``: (world, run_len, 2) gathered records (elite runs or top-m contributions)."""
        torch = _torch()
        world, run_len = runs.shape[0], runs.shape[1]
        cand = torch.empty(3 + self.p * (4 + self.D), dtype=torch.float64, device="cuda")
        nl = nat.c_int32(0)
        nat.check(self.lib.spasm_shard_descend(self.model.handle, self.model.dtype_id, ctypes_byref(self.cfg),
                                               restart, nat.ptr(runs.contiguous()), world, run_len, pos_lo, pos_hi,
                                               nat.ptr(self.warm), self.n_warm, nat.ptr(self.ws), self.ws.numel(),
                                               nat.ptr(cand), ctypes_byref(nl), nat.stream_handle()),
                  "shard_descend")
        self.launches += nl.value
        return cand


# the top-m select protocol replaces the all-gather of m records per rank once that gather
# exceeds this many bytes (below it, one collective beats the key_bits/8 + 2 small ones)
SELECT_PROTOCOL_BYTES = 4 << 20


def allot_top_m(counts: np.ndarray) -> np.ndarray:
    """Per-rank record counts of the global top m from the gathered (world, 3) rows
    (records below K*, records at K*, K* records the top m takes): every rank contributes
    its records below the threshold key and the K*-keyed ties go to the lowest global rows,
    i.e. to the lower ranks first (contiguous row shards)."""
    counts = np.asarray(counts, dtype=np.int64).reshape(-1, 3)
    less, ties, need = counts[:, 0], counts[:, 1], int(counts[0, 2])
    before = np.concatenate([[0], np.cumsum(ties)[:-1]])
    return less + np.clip(need - before, 0, ties)


def topm_exchange(ops, comm, restart: int, row_lo: int, n_local: int, m: int):
    """The exact distributed top-m selection of one restart (spasm_shard_topm_*): key_bits/8
    all-reduces of 256 counts, one all-gather of 3 counts, one all-gather of the rank's
    contribution (m records over all ranks). Returns (world, cap, 2) runs for descend."""
    ops.select(restart, row_lo, n_local, elite=False)
    st = ops.topm_init()
    for _ in range(ops.key_bits // 8):
        h = comm.all_reduce_sum(ops.topm_hist(st))
        ops.topm_pick(st, h)
    take = allot_top_m(comm.all_gather(ops.topm_local(st)).cpu().numpy())
    if int(take.sum()) != m:  # the ranks disagree on the threshold: a broken exchange, not a result
        raise RuntimeError(f"top-m select allotted {int(take.sum())} records for m = {m}: {take.tolist()}")
    cap = max(1, int(take.max()))
    return comm.all_gather(ops.topm_contrib(int(take[comm.rank]), cap)).reshape(comm.world, cap, 2)


def merge_candidates(blocks: np.ndarray, D: int, p_return: int, epsilon: float):
    """Host merge of the gathered candidate blocks (world, 3 + p*(4+D)).

    Returns (n_satisfying, flagged, rows) with rows = the first p_return satisfying
    records in the reference's stable order (quadratic cost, then position in the top-m
    order; particle_opt.py:360-365), after dropping those failing the re-check
    (particle_opt.py:366). Each row is (position, row, cost, recheck, values[D])."""
    blocks = np.asarray(blocks, dtype=float).reshape(blocks.shape[0], -1)
    n_sat = int(blocks[:, 0].sum())
    flagged = int(blocks[:, 1].sum())
    recs = []
    for b in blocks:
        k = int(b[2])
        recs.extend(b[3: 3 + k * (4 + D)].reshape(k, 4 + D))
    if not recs:
        return n_sat, flagged, np.zeros((0, 4 + D))
    recs = np.asarray(recs)
    order = np.lexsort((recs[:, 0], recs[:, 2]))[:p_return]
    chosen = recs[order]
    chosen = chosen[chosen[:, 3] < epsilon]
    return n_sat, flagged, chosen


def solve_sharded(cost_model, config: OptimizerConfig, *, group=None, comm=None, ops=None, warm_seeds=None,
                  sampler: str = "pcg64", protocol: str = "auto") -> SolveResult:
    """``particle_opt.solve`` (reference particle_opt.py:303-400) over all ranks of ``group``.

    Every rank must call it with the same model, config and warm seeds; every rank returns
    the same result. ``comm`` / ``ops`` override the collective and device halves (the CPU
    tests drive the host logic with a gloo group and oracle-backed halves)."""
    if sampler not in _SAMPLERS:
        raise ValueError(f"sampler must be one of {tuple(_SAMPLERS)}")
    comm = comm if comm is not None else TorchComm(group)
    t0 = time.perf_counter()
    D = cost_model.dimension
    warm = None
    if warm_seeds is not None:
        warm = np.atleast_2d(np.asarray(warm_seeds, dtype=float))
        if warm.shape[0] == 0:
            warm = None
        elif warm.shape[0] > config.n:
            raise ValueError("more seeds than particles")
        elif warm.shape[1] != D:
            raise ValueError("seed dimension mismatch")
    row_lo, row_hi = shard_range(config.n, comm.world, comm.rank)
    pos_lo, pos_hi = shard_range(config.m, comm.world, comm.rank)
    if ops is None:
        if not isinstance(cost_model, NativeCostModel):
            raise TypeError("solve_sharded needs a native cost model (problems.as_cost_model)")
        ops = NativeShardOps(cost_model, config, _SAMPLERS[sampler], warm, row_hi - row_lo, pos_hi - pos_lo)
    torch = _torch()
    dev0 = None
    if torch.cuda.is_available() and isinstance(ops, NativeShardOps):
        dev0 = torch.cuda.Event(enable_timing=True)
        dev0.record()
    steps = flagged_total = 0
    per = config.k_lin + config.k_quad
    result = None
    if protocol not in ("auto", "gather", "select"):
        raise ValueError("protocol must be 'auto', 'gather' or 'select'")
    use_select = protocol == "select" or (protocol == "auto" and comm.world > 1
                                          and comm.world * config.m * 16 > SELECT_PROTOCOL_BYTES)
    for restart in range(config.max_restarts):
        if use_select:
            runs = topm_exchange(ops, comm, restart, row_lo, row_hi - row_lo, config.m)
        else:
            elite = ops.select(restart, row_lo, row_hi - row_lo)
            runs = comm.all_gather(elite).reshape(comm.world, config.m, 2)
        cand = ops.descend(restart, runs, pos_lo, pos_hi)
        blocks = comm.all_gather(cand).cpu().numpy()
        steps += per
        n_sat, flagged, chosen = merge_candidates(blocks, D, config.p_return, config.epsilon)
        flagged_total += flagged
        if n_sat > 0:
            result = (restart, n_sat, chosen)
            break
    device_ms = None
    if dev0 is not None:
        dev1 = torch.cuda.Event(enable_timing=True)
        dev1.record()
        dev1.synchronize()
        device_ms = dev0.elapsed_time(dev1)
    launches = getattr(ops, "launches", 0)
    if result is None:
        report = SolveReport(restarts=config.max_restarts, steps=steps, time_ms=(time.perf_counter() - t0) * 1e3,
                             n_satisfying=0, flagged=flagged_total, device_ms=device_ms, launches=launches)
        return SolveResult(False, np.zeros((0, D)), np.zeros(0), np.zeros(0, dtype=np.int64), report)
    restart, n_sat, chosen = result
    report = SolveReport(restarts=restart, steps=steps, time_ms=(time.perf_counter() - t0) * 1e3, n_satisfying=n_sat,
                         flagged=flagged_total, device_ms=device_ms, launches=launches)
    return SolveResult(success=len(chosen) > 0, particles=chosen[:, 4:].copy(), costs=chosen[:, 2].copy(),
                       indices=chosen[:, 1].astype(np.int64), report=report)


__all__ = ["TorchComm", "NativeShardOps", "SELECT_PROTOCOL_BYTES", "allot_top_m", "merge_candidates", "shard_range",
           "solve_sharded", "topm_exchange", "torch_dtype"]
