"""Stage-1 particle engine on the B200: the reference's ``seqplace.particle_opt`` API
(reference particle_opt.py:33-400) with every numeric step on the GPU.

Two execution paths share the same semantics:

* native cost models (``TetrisCostModel`` / ``TowerCostModel`` from
  ``paper_2510_07674_b200.problems``) run the whole restart loop inside libspasm
  (``spasm_solve``): fused sample+evaluate, stable top-M radix sort, the fused
  K_lin+K_quad descent kernel, satisfying-particle ordering and the re-check, with one
  small device->host read per restart;
* any other ``CostModel`` whose ``evaluate``/``gradient`` accept and return CUDA
  tensors is driven from Python, with sampling, the clamped NaN-freezing step and the
  stable selection still done by libspasm kernels.

Determinism contract (reference particle_opt.py:14-18): sampling is one centralized
PCG64 stream per restart (bit-identical to numpy's draw), every per-particle
computation is row-independent and every ordering is a stable sort, so results do not
depend on the worker count (``threads`` is accepted and ignored) or GPU count.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as nat
from .geometry import LINEAR, QUADRATIC, _check_mode, mode_id

TRACE_PARTICLE_CAP = 4096

_PRECISIONS = {"fp32": nat.F32, "fp64": nat.F64}


def _torch():
    import torch

    return torch


def torch_dtype(precision: str):
    torch = _torch()
    return torch.float32 if precision == "fp32" else torch.float64


class CostModel:
    """Batch cost interface the engine optimizes against (reference particle_opt.py:33-61).

    ``evaluate(values (P, D), mode) -> (P,)`` and ``gradient(values, mode) -> (P, D)``.
    Models used with the Python-driven engine path must accept CUDA tensors.
    """

    precision = "fp64"

    def __init__(self, dimension: int, lower, upper):
        self.dimension = int(dimension)
        self.lower = np.asarray(lower, dtype=float)
        self.upper = np.asarray(upper, dtype=float)
        if self.lower.shape != (self.dimension,) or self.upper.shape != (self.dimension,):
            raise ValueError("bounds must have shape (dimension,)")
        if np.any(self.lower > self.upper):
            raise ValueError("lower bound exceeds upper bound")
        self._dev_bounds = {}

    def evaluate(self, values, mode: str):
        raise NotImplementedError

    def gradient(self, values, mode: str):
        raise NotImplementedError

    def satisfaction(self, values, epsilon: float = 1e-3):
        return self.evaluate(values, QUADRATIC) < epsilon

    def clamp(self, values):
        if isinstance(values, np.ndarray):
            return np.clip(values, self.lower, self.upper)
        lo, hi = self.device_bounds(values.dtype, values.device)
        return _torch().maximum(_torch().minimum(values, hi), lo)

    # device copies of the bounds, per (dtype, device)
    def device_bounds(self, dtype, device):
        key = (dtype, str(device))
        if key not in self._dev_bounds:
            torch = _torch()
            self._dev_bounds[key] = (
                torch.as_tensor(self.lower, dtype=dtype, device=device),
                torch.as_tensor(self.upper, dtype=dtype, device=device),
            )
        return self._dev_bounds[key]


class NativeCostModel(CostModel):
    """A cost model whose evaluate/gradient are libspasm kernels (C-ABI handle).

    Accepts numpy arrays (returns float64 numpy, H2D/D2H inside the call, the
    reference's calling convention) or CUDA tensors (returns CUDA tensors).
    ``precision`` is "fp32" (perf path) or "fp64" (parity path).
    """

    def __init__(self, dimension: int, lower, upper, handle, precision: str = "fp32"):
        super().__init__(dimension, lower, upper)
        if precision not in _PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(_PRECISIONS)}")
        self.precision = precision
        self._handle = handle
        self._lib = nat.load()

    @property
    def dtype_id(self) -> int:
        return _PRECISIONS[self.precision]

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and getattr(self, "_lib", None) is not None:
            self._lib.spasm_model_destroy(h)
            self._handle = None

    def _prep(self, values):
        torch = _torch()
        nat.require_cuda()
        is_np = not isinstance(values, torch.Tensor)
        dt = torch_dtype(self.precision)
        if is_np:
            arr = np.asarray(values, dtype=float)
            if arr.ndim != 2 or arr.shape[1] != self.dimension:
                raise ValueError(f"values must have shape (P, {self.dimension})")
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(device="cuda", dtype=dt)
        else:
            if values.ndim != 2 or values.shape[1] != self.dimension:
                raise ValueError(f"values must have shape (P, {self.dimension})")
            t = values.to(device="cuda", dtype=dt).contiguous()
        return t, is_np

    def evaluate(self, values, mode: str):
        _check_mode(mode)
        t, is_np = self._prep(values)
        out = _torch().empty(t.shape[0], dtype=t.dtype, device=t.device)
        nat.check(self._lib.spasm_evaluate(self._handle, self.dtype_id, nat.ptr(t), t.shape[0], mode_id(mode),
                                           nat.ptr(out), nat.stream_handle()), "evaluate")
        return out.double().cpu().numpy() if is_np else out

    def gradient(self, values, mode: str):
        _check_mode(mode)
        t, is_np = self._prep(values)
        out = _torch().empty_like(t)
        nat.check(self._lib.spasm_gradient(self._handle, self.dtype_id, nat.ptr(t), t.shape[0], mode_id(mode),
                                           nat.ptr(out), nat.stream_handle()), "gradient")
        return out.double().cpu().numpy() if is_np else out


@dataclass
class ParticleBatch:
    """Matrix of candidate solutions plus their evaluated costs (numpy or CUDA tensors)."""

    values: object
    costs: object
    satisfied: object = field(default=None)
    flagged: object = field(default=None)

    def __post_init__(self):
        torch = _torch()
        if isinstance(self.values, torch.Tensor):
            n = self.values.shape[0]
            dev = self.values.device
            if not isinstance(self.costs, torch.Tensor):
                self.costs = torch.as_tensor(np.asarray(self.costs, dtype=float), device=dev,
                                             dtype=self.values.dtype)
            if self.satisfied is None:
                self.satisfied = torch.zeros(n, dtype=torch.bool, device=dev)
            if self.flagged is None:
                self.flagged = torch.zeros(n, dtype=torch.bool, device=dev)
        else:
            self.values = np.asarray(self.values, dtype=float)
            self.costs = np.asarray(self.costs, dtype=float)
            n = len(self.values)
            if self.satisfied is None:
                self.satisfied = np.zeros(n, dtype=bool)
            if self.flagged is None:
                self.flagged = np.zeros(n, dtype=bool)

    def __len__(self) -> int:
        return int(self.values.shape[0])


@dataclass
class OptimizerConfig:
    """Engine hyperparameters (reference particle_opt.py:86-113, same defaults/validation)."""

    n: int = 4096
    m: int = 512
    k_lin: int = 25
    k_quad: int = 5
    eta_init: float = 0.1
    alpha: float = 0.05
    epsilon: float = 1e-3
    p_return: int = 32
    max_restarts: int = 64
    seed: int = 0
    # perf-mode particle update (north_star item 4; not in the reference, whose defaults
    # these keep): "adam" scales Adam moments by the same learning-rate schedule;
    # noise_sigma > 0 adds Gaussian noise (std = noise_sigma x bound width, Philox stream)
    # annealed linearly to 0 over the K_lin linear steps
    update: str = "gd"
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    noise_sigma: float = 0.0

    def __post_init__(self):
        if not (1 <= self.m <= self.n):
            raise ValueError("need 1 <= m <= n")
        if self.k_lin < 0 or self.k_quad < 0:
            raise ValueError("step counts must be nonnegative")
        if self.eta_init <= 0 or self.alpha <= 0:
            raise ValueError("learning rates must be positive")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.p_return < 1:
            raise ValueError("p_return must be >= 1")
        if self.max_restarts < 1:
            raise ValueError("max_restarts must be >= 1")
        if self.update not in ("gd", "adam"):
            raise ValueError("update must be 'gd' or 'adam'")
        if self.noise_sigma < 0:
            raise ValueError("noise_sigma must be >= 0")
        if self.update == "adam" and not (0 <= self.adam_beta1 < 1 and 0 <= self.adam_beta2 < 1 and self.adam_eps > 0):
            raise ValueError("Adam needs 0 <= beta1, beta2 < 1 and eps > 0")

    @property
    def reference_update(self) -> bool:
        """True when the particle update is the reference's clamped gradient step."""
        return self.update == "gd" and self.noise_sigma == 0.0

    def native(self, sampler: int, n_traced: int = 0):
        """The spasm_solve_config C struct of this configuration."""
        return nat.spasm_solve_config(self.n, self.m, self.k_lin, self.k_quad, self.eta_init, self.alpha,
                                      self.epsilon, self.p_return, self.max_restarts, self.seed, sampler, n_traced,
                                      1 if self.update == "adam" else 0, self.adam_beta1, self.adam_beta2,
                                      self.adam_eps, self.noise_sigma)


@dataclass
class TraceData:
    steps: np.ndarray
    particle_ids: np.ndarray
    selected: np.ndarray
    costs: np.ndarray
    satisfied: np.ndarray


@dataclass
class SolveReport:
    restarts: int
    steps: int
    time_ms: float
    n_satisfying: int = 0
    flagged: int = 0
    trace: Optional[TraceData] = None
    device_ms: Optional[float] = None
    launches: int = 0  # libspasm kernels launched (native path)


@dataclass
class SolveResult:
    success: bool
    particles: np.ndarray
    costs: np.ndarray
    indices: np.ndarray
    report: SolveReport


# ---------------------------------------------------------------------------
# restart streams and sampling
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class RestartStream:
    """Device stand-in for ``restart_stream(seed, restart)`` (particle_opt.py:176-178).

    Draws are bit-identical to numpy's ``default_rng(SeedSequence(seed, spawn_key=(restart,)))``
    stream: the PCG64 state is derived by libspasm's SeedSequence restatement and
    each particle row jumps ahead to its slice of the stream on the device.
    ``row_offset`` selects a contiguous shard of the rows of one centralized draw.
    """

    seed: int
    restart: int
    sampler: int = nat.SAMPLER_PCG64
    row_offset: int = 0

    def pcg64_state(self) -> tuple[int, int]:
        out = (nat.c_uint64 * 4)()
        nat.check(nat.load().spasm_pcg64_state(self.seed, self.restart, out), "pcg64_state")
        return (out[0] << 64) | out[1], (out[2] << 64) | out[3]

    def uniform(self, lower, upper, size, *, dtype=None, warm=None):
        """(size[0], D) uniform draw on the device (CUDA tensor)."""
        torch = _torch()
        nat.require_cuda()
        n, d = int(size[0]), int(size[1])
        lo = np.ascontiguousarray(np.broadcast_to(np.asarray(lower, dtype=float), (d,)))
        hi = np.ascontiguousarray(np.broadcast_to(np.asarray(upper, dtype=float), (d,)))
        dt = dtype or torch.float64
        out = torch.empty((n, d), dtype=dt, device="cuda")
        wt = None
        nw = 0
        if warm is not None and len(warm):
            wt = torch.as_tensor(np.ascontiguousarray(warm, dtype=float), device="cuda")
            nw = wt.shape[0]
        did = nat.F32 if dt == torch.float32 else nat.F64
        nat.check(nat.load().spasm_sample(did, d, nat.ptr(lo), nat.ptr(hi), self.seed, self.restart, self.sampler,
                                          self.row_offset, n, nat.ptr(wt), nw, nat.ptr(out), nat.stream_handle()),
                  "sample")
        return out


def restart_stream(seed: int, restart: int) -> RestartStream:
    """RNG stream for one restart, keyed by (seed, restart index)."""
    return RestartStream(int(seed), int(restart))


def _value_dtype(cost_model):
    return torch_dtype(getattr(cost_model, "precision", "fp64"))


def sample_uniform(cost_model: CostModel, n: int, rng_stream: RestartStream) -> ParticleBatch:
    """n i.i.d. uniform particles within the model's bounds (particle_opt.py:181-192)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    torch = _torch()
    values = rng_stream.uniform(cost_model.lower, cost_model.upper, (n, cost_model.dimension),
                                dtype=_value_dtype(cost_model))
    return ParticleBatch(values=values, costs=torch.full((n,), float("inf"), dtype=values.dtype, device=values.device))


def _sort_indices(costs_t, m: int):
    """Stable ascending order of a CUDA cost vector, first m indices (int64 tensor)."""
    torch = _torch()
    lib = nat.load()
    n = costs_t.shape[0]
    did = nat.F32 if costs_t.dtype == torch.float32 else nat.F64
    kdt = torch.int32 if did == nat.F32 else torch.int64
    keys = torch.empty(n, dtype=kdt, device=costs_t.device)
    vals = torch.empty(n, dtype=torch.int32, device=costs_t.device)
    nb = torch.zeros(1, dtype=torch.int32, device=costs_t.device)
    s = nat.stream_handle()
    nat.check(lib.spasm_cost_keys(did, nat.ptr(costs_t.contiguous()), n, float("inf"), nat.ptr(keys), nat.ptr(vals),
                                  nat.ptr(nb), s), "cost_keys")
    ws = torch.empty(max(1, lib.spasm_sort_workspace_bytes(did, n)), dtype=torch.uint8, device=costs_t.device)
    nat.check(lib.spasm_sort_pairs(did, nat.ptr(keys), nat.ptr(vals), n, nat.ptr(ws), s), "sort")
    return vals[:m].long()


def select_topk(batch: ParticleBatch, m: int):
    """Indices of the m lowest-cost particles, ascending, ties by row index (particle_opt.py:195-200)."""
    if m > len(batch):
        raise ValueError("m exceeds batch size")
    torch = _torch()
    nat.require_cuda()
    if isinstance(batch.costs, torch.Tensor):
        return _sort_indices(batch.costs.cuda(), m)
    c = torch.as_tensor(np.asarray(batch.costs, dtype=float), device="cuda")
    return _sort_indices(c, m).cpu().numpy()


def lr_schedule(k: int, k_lin: int, eta_init: float) -> float:
    """Linear decay eta_init * (1 - k/K_lin) for k in 1..K_lin (particle_opt.py:203-211)."""
    if not 1 <= k <= k_lin:
        raise ValueError("schedule step k out of range 1..k_lin")
    return eta_init * (1.0 - k / k_lin)


def _as_device(values, dtype):
    torch = _torch()
    if isinstance(values, torch.Tensor):
        return values.to(device="cuda", dtype=dtype).contiguous(), False
    return torch.as_tensor(np.ascontiguousarray(values, dtype=float), device="cuda").to(dtype), True


def _step_values(values_t, flagged_t, model: CostModel, mode: str, rate: float) -> None:
    """One clamped gradient step in place with the NaN freeze (particle_opt.py:214-228)."""
    torch = _torch()
    grad = model.gradient(values_t, mode)
    if not isinstance(grad, torch.Tensor):
        grad = torch.as_tensor(np.asarray(grad, dtype=float), device=values_t.device)
    grad = grad.to(values_t.dtype).contiguous()
    lo, hi = model.device_bounds(values_t.dtype, values_t.device)
    did = nat.F32 if values_t.dtype == torch.float32 else nat.F64
    fl = torch.zeros(values_t.shape[0], dtype=torch.uint8, device=values_t.device)
    nat.check(nat.load().spasm_step(did, nat.ptr(values_t), nat.ptr(grad), values_t.shape[0], values_t.shape[1],
                                    float(rate), nat.ptr(lo), nat.ptr(hi), nat.ptr(fl), nat.stream_handle()), "step")
    flagged_t |= fl.bool()


def _eval_t(model, values_t, mode):
    torch = _torch()
    c = model.evaluate(values_t, mode)
    if not isinstance(c, torch.Tensor):
        c = torch.as_tensor(np.asarray(c, dtype=float), device=values_t.device)
    return c


def descend(batch: ParticleBatch, cost_model: CostModel, mode: str, rate: float, threads: int = 1) -> ParticleBatch:
    """One clamped gradient step on every particle, costs re-evaluated (particle_opt.py:231-247)."""
    if rate < 0:
        raise ValueError("rate must be >= 0")
    torch = _torch()
    nat.require_cuda()
    vt, was_np = _as_device(batch.values, _value_dtype(cost_model))
    ft = torch.as_tensor(np.asarray(batch.flagged), device="cuda") if was_np else batch.flagged.cuda()
    _step_values(vt, ft, cost_model, mode, rate)
    ct = _eval_t(cost_model, vt, mode)
    if was_np:
        batch.values[...] = vt.double().cpu().numpy()
        batch.flagged[...] = ft.cpu().numpy()
        batch.costs = ct.double().cpu().numpy()
    else:
        batch.values.copy_(vt)
        batch.flagged.copy_(ft)
        batch.costs = ct
    return batch


def inject_warm_start(batch: ParticleBatch, seeds, cost_model: CostModel) -> ParticleBatch:
    """Overwrite the first rows with clamped seed states (particle_opt.py:250-263)."""
    seeds = np.atleast_2d(np.asarray(seeds, dtype=float))
    if seeds.shape[0] == 0:
        return batch
    if seeds.shape[0] > len(batch):
        raise ValueError("more seeds than particles")
    if seeds.shape[1] != cost_model.dimension:
        raise ValueError("seed dimension mismatch")
    clamped = np.clip(seeds, cost_model.lower, cost_model.upper)
    torch = _torch()
    k = seeds.shape[0]
    if isinstance(batch.values, torch.Tensor):
        batch.values[:k] = torch.as_tensor(clamped, device=batch.values.device).to(batch.values.dtype)
        batch.costs[:k] = float("inf")
    else:
        batch.values[:k] = clamped
        batch.costs[:k] = np.inf
    return batch


def run_descent_schedule(model: CostModel, values, config: OptimizerConfig, *, threads: int = 1, trace_sink=None,
                         epsilon: Optional[float] = None):
    """K_lin linear steps with the decaying rate, then K_quad quadratic steps at alpha
    (particle_opt.py:266-300). Returns (values, flagged, steps); values updated in place.

    Native models without a trace sink run the whole schedule as one fused kernel.
    """
    torch = _torch()
    nat.require_cuda()
    eps = config.epsilon if epsilon is None else epsilon
    vt, was_np = _as_device(values, _value_dtype(model))
    P = vt.shape[0]
    steps = config.k_lin + config.k_quad
    if isinstance(model, NativeCostModel) and trace_sink is None:
        out_v = torch.empty_like(vt)
        out_c = torch.empty(P, dtype=vt.dtype, device=vt.device)
        fl = torch.zeros(P, dtype=torch.uint8, device=vt.device)
        nat.check(nat.load().spasm_descent_schedule(
            model.handle, model.dtype_id, nat.ptr(vt), None, P, config.k_lin, config.k_quad, config.eta_init,
            config.alpha, eps, nat.ptr(out_v), nat.ptr(out_c), nat.ptr(fl), None, None, None, 0,
            nat.stream_handle()), "descent_schedule")
        vt.copy_(out_v)
        flagged = fl.bool()
    else:
        flagged = torch.zeros(P, dtype=torch.bool, device=vt.device)
        step = 0
        for k in range(1, config.k_lin + 1):
            _step_values(vt, flagged, model, LINEAR, lr_schedule(k, config.k_lin, config.eta_init))
            step += 1
            if trace_sink is not None:
                trace_sink(step, LINEAR, _eval_t(model, vt, LINEAR), _eval_t(model, vt, QUADRATIC) < eps)
        for _ in range(config.k_quad):
            _step_values(vt, flagged, model, QUADRATIC, config.alpha)
            step += 1
            if trace_sink is not None:
                cq = _eval_t(model, vt, QUADRATIC)
                trace_sink(step, QUADRATIC, cq, cq < eps)
    if was_np:
        values[...] = vt.double().cpu().numpy()
        return values, flagged.cpu().numpy(), steps
    if vt.data_ptr() != values.data_ptr():
        values.copy_(vt)
    return values, flagged, steps


# ---------------------------------------------------------------------------
# solve
# ---------------------------------------------------------------------------

_SAMPLERS = {"pcg64": nat.SAMPLER_PCG64, "philox": nat.SAMPLER_PHILOX}


def solve(cost_model: CostModel, config: OptimizerConfig, *, warm_seeds=None, threads: int = 1, trace: bool = False,
          sampler: str = "pcg64") -> SolveResult:
    """Full sample / select / optimize / extract loop with restarts (particle_opt.py:303-400).

    Returns up to ``p_return`` satisfying particles ordered by ascending quadratic cost;
    failure after ``max_restarts`` attempts is a normal return with ``success=False``.
    ``sampler="philox"`` switches the initial draw to the perf-mode counter stream
    (not bit-compatible with the reference's numpy streams).
    """
    if sampler not in _SAMPLERS:
        raise ValueError(f"sampler must be one of {tuple(_SAMPLERS)}")
    nat.require_cuda()
    if isinstance(cost_model, NativeCostModel):
        return _solve_native(cost_model, config, warm_seeds, trace, _SAMPLERS[sampler])
    if not config.reference_update:
        raise ValueError("update='adam' / noise_sigma > 0 run inside the native kernels: use a native cost model")
    return _solve_generic(cost_model, config, warm_seeds, trace, _SAMPLERS[sampler])


class _Workspace:
    """Device scratch for ``spasm_solve``, keyed by what sizes it (dtype, D, n, m, p_return,
    n_warm, device) -- not by the model: the buffer is plain scratch, so the C4 replanning
    loop's per-tick models share one entry instead of leaving one per dead model behind.
    At most ``cap`` entries are kept (least recently used dropped). A model's cached CUDA
    graph records the workspace pointer and is re-captured if it changes (capi.cu)."""

    def __init__(self, cap: int = 8):
        self._cache = {}
        self._cap = cap

    def get(self, model: NativeCostModel, cfg, n_warm: int):
        torch = _torch()
        key = (model.dtype_id, model.dimension, cfg.n, cfg.m, cfg.p_return, n_warm, torch.cuda.current_device())
        nbytes = nat.load().spasm_solve_workspace_bytes(model.handle, model.dtype_id, ctypes_byref(cfg), n_warm)
        buf = self._cache.pop(key, None)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self._cache[key] = buf  # most recently used last
        while len(self._cache) > self._cap:
            self._cache.pop(next(iter(self._cache)))
        return buf


def ctypes_byref(x):
    import ctypes

    return ctypes.byref(x)


_WS = _Workspace()


def _warm_rows(warm_seeds, config, D):
    if warm_seeds is None:
        return None, 0
    warm = np.atleast_2d(np.asarray(warm_seeds, dtype=float))
    if warm.shape[0] == 0:
        return None, 0
    if warm.shape[0] > config.n:
        raise ValueError("more seeds than particles")
    if warm.shape[1] != D:
        raise ValueError("seed dimension mismatch")
    return np.ascontiguousarray(warm), warm.shape[0]


class PendingSolve:
    """A stage-1 solve launched on the device and not yet read back (``solve_launch``).

    With a repeated shape the whole restart loop is one CUDA graph launch (a conditional
    WHILE node; the success test runs on the device), so nothing waits for the host until
    ``collect``. ``device_rows`` exposes the compacted result rows in device memory, so a
    stage-2 consumer can read them in stream order without a round trip."""

    def __init__(self, model, config, t0, warm, workspace):
        self.model, self.config, self.t0 = model, config, t0
        self._warm = warm  # kept alive until the launch has copied it
        self._ws = workspace  # the device rows live in it: kept alive until collect (cache eviction)

    def device_rows(self):
        """(rows pointer: float64 (p_return, D), count pointer: int32) on the device."""
        rows = nat.c_void_p()
        count = nat.c_void_p()
        nat.check(nat.load().spasm_solve_device_rows(self.model.handle, nat.byref(rows), nat.byref(count)),
                  "solve_device_rows")
        return rows.value, count.value

    def collect(self) -> "SolveResult":
        config, D = self.config, self.model.dimension
        parts = np.zeros((config.p_return, D))
        costs = np.zeros(config.p_return)
        idx = np.zeros(config.p_return, dtype=np.int64)
        rep = nat.spasm_solve_report()
        status = nat.check(nat.load().spasm_solve_collect(self.model.handle, nat.ptr(parts), nat.ptr(costs),
                                                          nat.ptr(idx), ctypes_byref(rep)), "solve_collect")
        self._ws = None
        return _result(status, rep, parts, costs, idx, self.t0, None)


def _result(status, rep, parts, costs, idx, t0, trace_data):
    k = int(rep.n_chosen) if status == nat.SPASM_OK else 0
    report = SolveReport(
        restarts=int(rep.restarts),
        steps=int(rep.steps),
        time_ms=(time.perf_counter() - t0) * 1e3,
        n_satisfying=int(rep.n_satisfying),
        flagged=int(rep.flagged),
        trace=trace_data,
        device_ms=float(rep.device_ms),
        launches=int(rep.launches),
    )
    return SolveResult(success=bool(rep.success), particles=parts[:k].copy(), costs=costs[:k].copy(),
                       indices=idx[:k].copy(), report=report)


def solve_launch(model: NativeCostModel, config: OptimizerConfig, *, warm_seeds=None,
                 sampler: str = "pcg64") -> PendingSolve:
    """Start ``solve`` on the device and return without waiting (see PendingSolve)."""
    if sampler not in _SAMPLERS:
        raise ValueError(f"sampler must be one of {tuple(_SAMPLERS)}")
    nat.require_cuda()
    if not isinstance(model, NativeCostModel):
        raise TypeError("solve_launch needs a native cost model")
    t0 = time.perf_counter()
    warm, n_warm = _warm_rows(warm_seeds, config, model.dimension)
    cfg = config.native(_SAMPLERS[sampler], 0)
    ws = _WS.get(model, cfg, n_warm)
    nat.check(nat.load().spasm_solve_launch(model.handle, model.dtype_id, ctypes_byref(cfg), nat.ptr(warm), n_warm,
                                            nat.ptr(ws), ws.numel(), nat.stream_handle()), "solve_launch")
    return PendingSolve(model, config, t0, warm, ws)


def _solve_native(model: NativeCostModel, config: OptimizerConfig, warm_seeds, trace: bool, sampler: int):
    torch = _torch()
    t0 = time.perf_counter()
    D = model.dimension
    warm, n_warm = _warm_rows(warm_seeds, config, D)
    n_traced = min(config.m, TRACE_PARTICLE_CAP) if trace else 0
    cfg = config.native(sampler, n_traced)
    ws = _WS.get(model, cfg, n_warm)
    parts = np.zeros((config.p_return, D))
    costs = np.zeros(config.p_return)
    idx = np.zeros(config.p_return, dtype=np.int64)
    rep = nat.spasm_solve_report()
    steps_total = config.k_lin + config.k_quad
    tc = ts = tid = None
    if n_traced:
        tc = torch.zeros((steps_total, n_traced), dtype=torch_dtype(model.precision), device="cuda")
        ts = torch.zeros((steps_total, n_traced), dtype=torch.uint8, device="cuda")
        tid = torch.zeros(n_traced, dtype=torch.int32, device="cuda")
    status = nat.check(nat.load().spasm_solve(model.handle, model.dtype_id, ctypes_byref(cfg), nat.ptr(warm), n_warm,
                                              nat.ptr(ws), ws.numel(), nat.ptr(parts), nat.ptr(costs), nat.ptr(idx),
                                              ctypes_byref(rep), nat.ptr(tc), nat.ptr(ts), nat.ptr(tid),
                                              nat.stream_handle()), "solve")
    trace_data = None
    if n_traced:
        trace_data = TraceData(
            steps=np.arange(1, steps_total + 1),
            particle_ids=tid.cpu().numpy().astype(np.int64),
            selected=np.ones(n_traced, dtype=bool),
            costs=tc.double().cpu().numpy(),
            satisfied=ts.cpu().numpy().astype(bool),
        )
    return _result(status, rep, parts, costs, idx, t0, trace_data)


def _solve_generic(model: CostModel, config: OptimizerConfig, warm_seeds, trace: bool, sampler: int):
    """Python-driven restart loop for cost models that evaluate CUDA tensors themselves."""
    torch = _torch()
    t0 = time.perf_counter()
    total_steps = 0
    total_flagged = 0
    trace_data = None
    dt = _value_dtype(model)
    for restart in range(config.max_restarts):
        rng = RestartStream(int(config.seed), restart, sampler)
        batch = sample_uniform(model, config.n, rng)
        if warm_seeds is not None:
            inject_warm_start(batch, warm_seeds, model)
        batch.costs = _eval_t(model, batch.values, LINEAR).to(dt)
        top = select_topk(batch, config.m)
        values = batch.values[top].contiguous()

        sink = None
        if trace:
            n_traced = min(config.m, TRACE_PARTICLE_CAP)
            step_count = config.k_lin + config.k_quad
            t_costs = np.zeros((step_count, n_traced))
            t_sat = np.zeros((step_count, n_traced), dtype=bool)

            def sink(step, mode, costs, satisfied, _c=t_costs, _s=t_sat, _n=n_traced):
                _c[step - 1] = costs[:_n].double().cpu().numpy()
                _s[step - 1] = satisfied[:_n].cpu().numpy()

            trace_data = TraceData(steps=np.arange(1, step_count + 1), particle_ids=top[:n_traced].cpu().numpy(),
                                   selected=np.ones(n_traced, dtype=bool), costs=t_costs, satisfied=t_sat)

        values, flagged, steps = run_descent_schedule(model, values, config, trace_sink=sink)
        total_steps += steps
        total_flagged += int(flagged.sum().item())
        final_costs = _eval_t(model, values, QUADRATIC).to(dt)
        sat = final_costs < config.epsilon
        n_sat = int(sat.sum().item())
        if n_sat:
            sat_idx = torch.nonzero(sat).flatten()
            order = sat_idx[_sort_indices(final_costs[sat_idx].contiguous(), n_sat)]
            chosen = order[: config.p_return]
            recheck = model.satisfaction(values[chosen], config.epsilon)
            if not isinstance(recheck, torch.Tensor):
                recheck = torch.as_tensor(np.asarray(recheck), device=values.device)
            chosen = chosen[recheck.bool()]
            report = SolveReport(restarts=restart, steps=total_steps, time_ms=(time.perf_counter() - t0) * 1e3,
                                 n_satisfying=n_sat, flagged=total_flagged, trace=trace_data)
            return SolveResult(success=len(chosen) > 0, particles=values[chosen].double().cpu().numpy(),
                               costs=final_costs[chosen].double().cpu().numpy(),
                               indices=top[chosen].cpu().numpy().astype(np.int64), report=report)
    report = SolveReport(restarts=config.max_restarts, steps=total_steps, time_ms=(time.perf_counter() - t0) * 1e3,
                         n_satisfying=0, flagged=total_flagged, trace=trace_data)
    return SolveResult(success=False, particles=np.zeros((0, model.dimension)), costs=np.zeros(0),
                       indices=np.zeros(0, dtype=np.int64), report=report)
