"""Drop the B200 path into an installed reference package (``seqplace``) by rebinding the
hot-path names its ``bench`` module binds at import (reference bench.py:28-51), so every
caller -- ``solve_scene``, ``run_trials``, ``run_sweep``, the CLI -- runs on the GPU:

    import seqplace.bench
    from paper_2510_07674_b200.dropin import enable
    enable(seqplace.bench, precision="fp32")

The reference's objects (problems, chains, grasps, configs) are converted field by field into
this package's dataclasses, which mirror them name for name (the conversion is by the target
dataclass's fields, so nothing reference-specific is hard-coded), and this package's
``LiftFailure`` / ``TrajOptFailure`` are re-raised as the reference's own classes so its
``except`` clauses (bench.py:237-246) still catch them. Results are returned as this
package's dataclasses, which carry the same attribute names the reference reads.
"""
from __future__ import annotations

import dataclasses
import functools

from . import geometry, particle_opt, robot, trajopt
from . import problems as _problems

_OURS = {}
for _mod in (geometry, robot, trajopt, particle_opt, _problems):
    for _name in dir(_mod):
        _obj = getattr(_mod, _name)
        if isinstance(_obj, type) and dataclasses.is_dataclass(_obj):
            _OURS.setdefault(_name, _obj)


def to_native(obj):
    """A reference dataclass instance (or a list / tuple / dict of them) as this package's
    dataclass of the same name; anything else is returned unchanged."""
    if isinstance(obj, (list, tuple)):
        return type(obj)(to_native(v) for v in obj)
    if isinstance(obj, dict):
        return {k: to_native(v) for k, v in obj.items()}
    if not dataclasses.is_dataclass(obj) or isinstance(obj, type):
        return obj
    cls = _OURS.get(type(obj).__name__)
    if cls is None or isinstance(obj, cls):
        return obj
    kw = {f.name: to_native(getattr(obj, f.name)) for f in dataclasses.fields(cls) if f.init and hasattr(obj, f.name)}
    out = cls.__new__(cls)
    # frozen dataclasses with validating __post_init__ (they re-check what the reference
    # already checked) are built through __init__ so derived fields are recomputed
    out.__init__(**kw)
    return out


def _adapt(fn, ref_bench):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        args = tuple(to_native(a) for a in args)
        kwargs = {k: to_native(v) for k, v in kwargs.items()}
        try:
            return fn(*args, **kwargs)
        except trajopt.TrajOptFailure as exc:
            raise ref_bench.TrajOptFailure(exc.best_violation, exc.report) from exc
        except trajopt.LiftFailure as exc:
            raise ref_bench.LiftFailure(str(exc)) from exc

    return call


def enable(ref_bench, precision: str = "fp32"):
    """Rebind ``ref_bench`` (the reference's ``seqplace.bench`` module) onto the GPU path.
    Returns the previous bindings (pass them to ``disable`` to undo)."""
    names = ("as_cost_model", "solve", "lift_placements", "init_trajectories", "solve_al", "validate",
             "motion_endpoints", "trajectory_path_length")
    previous = {n: getattr(ref_bench, n) for n in names}
    ref_bench.as_cost_model = _adapt(functools.partial(_problems.as_cost_model, precision=precision), ref_bench)
    ref_bench.solve = _adapt(particle_opt.solve, ref_bench)
    for n in names[2:]:
        fn = getattr(trajopt, n)
        if n == "validate":
            fn = functools.partial(fn, precision="fp64")  # the independent re-check stays float64
        setattr(ref_bench, n, _adapt(fn, ref_bench))
    return previous


def disable(ref_bench, previous):
    for n, fn in previous.items():
        setattr(ref_bench, n, fn)
