"""Register the B200 backend inside an UNMODIFIED reference ``densolve`` install.

This is INTEGRATION.md §2 done at run time instead of by editing the reference's
files: ``install(densolve)`` adds ``"b200"`` to ``densolve.backends.BACKEND_NAMES``
and ``get_backend`` (backends.py:255-264), and puts a dispatch in front of the
reference's solver entry points (krylov.py:36/75/185 ``cg_solve`` / ``gmres_solve`` /
``bicgstab_solve``, direct.py:25/50/87/155/166 ``lu_factor_unblocked`` /
``lu_factor_blocked`` / ``cholesky_factor`` / ``lu_solve`` / ``cholesky_solve``,
direct.py:123/139 the substitutions): a call whose backend is the B200 one runs the
fused device solver of this package, every other call runs the reference unchanged.
Results come back as the reference's own ``SolveReport`` / ``LuFactors`` types and
errors as the reference's own exception classes (core.py:17-42), so the reference's
CLI, ``run_benchmark`` and tests drive the B200 path by backend name.

``fused=False`` keeps the reference's solver bodies and only swaps the backend: the
Python loops of krylov.py / direct.py then call the B200 op contract
(``ds_gemv``, ``ds_dot`` ...) one operation at a time.
"""

from __future__ import annotations

import dataclasses
import functools
import sys

from . import core, direct, krylov
from .backends import B200Backend

# (module, function, position of the backend argument or None, ours)
_SOLVERS = (
    ("krylov", "cg_solve", 4, krylov.cg_solve),
    ("krylov", "gmres_solve", 4, krylov.gmres_solve),
    ("krylov", "bicgstab_solve", 4, krylov.bicgstab_solve),
    ("direct", "lu_factor_blocked", 2, direct.lu_factor_blocked),
    ("direct", "lu_factor_unblocked", 1, direct.lu_factor_unblocked),
    ("direct", "cholesky_factor", 2, direct.cholesky_factor),
)
# no backend argument: dispatch on the factor object (ours carries a device handle)
_FACTOR_SOLVES = (("direct", "lu_solve", direct.lu_solve), ("direct", "cholesky_solve", direct.cholesky_solve))

_ERRORS = ("DimensionError", "PrecisionError", "DegenerateRhsError", "SingularMatrixError", "NotSpdError",
           "LinAlgError")


class _Translate:
    """Re-raise this package's exceptions as the reference's classes (same message)."""

    def __init__(self, ref):
        self.ref = ref

    def __enter__(self):
        return self

    def __exit__(self, et, ev, tb):
        if et is None or not issubclass(et, core.LinAlgError):
            return False
        for name in _ERRORS:
            if isinstance(ev, getattr(core, name)):
                cls = getattr(self.ref.core, name)
                err = cls(str(ev), getattr(ev, "index", None)) if name == "NotSpdError" else cls(str(ev))
                raise err from ev
        return False


def _to_ref(ref, obj):
    """Our SolveReport / LuFactors / CholeskyFactor -> the reference dataclass of the same
    name (field for field); the device handle rides along as an attribute."""
    for ours, name in ((core.SolveReport, "SolveReport"), (core.LuFactors, "LuFactors")):
        if isinstance(obj, ours):
            cls = getattr(ref.core, name)
            names = {f.name for f in dataclasses.fields(cls)}
            out = cls(**{f.name: getattr(obj, f.name) for f in dataclasses.fields(obj) if f.name in names})
            if getattr(obj, "device", None) is not None:
                out._b200 = obj
            return out
    if isinstance(obj, core.CholeskyFactor):
        cls = getattr(ref.core, "CholeskyFactor", None)
        if cls is not None:
            out = cls(l=obj.l)
            out._b200 = obj
            return out
    return obj


def _convert_result(ref, res):
    if isinstance(res, tuple):
        return tuple(_to_ref(ref, r) for r in res)
    return _to_ref(ref, res)


def backend_class(ref):
    """A B200Backend that IS a reference Backend (isinstance checks, name "b200") and
    raises the reference's exception classes from its ops."""
    ops = ("axpy", "dot", "nrm2", "scal", "iamax", "gemv", "ger", "gemm", "trsm_lower_unit", "trsm_upper")

    def wrap(name):
        base = getattr(B200Backend, name)

        @functools.wraps(base)
        def op(self, *a, **k):
            with _Translate(ref):
                return base(self, *a, **k)
        return op

    body = {name: wrap(name) for name in ops}
    body["__init__"] = lambda self, device=None, **_ignored: B200Backend.__init__(self, device)
    body["__doc__"] = "B200Backend registered in the reference (plugin.install)."
    return type("B200Backend", (B200Backend, ref.backends.Backend), body)


def _is_b200(be) -> bool:
    return isinstance(be, B200Backend)


def install(ref=None, fused: bool = True):
    """Register "b200" in the reference package ``ref`` (default: ``import densolve``).
    Idempotent; returns the backend class."""
    if ref is None:
        import densolve as ref  # noqa: PLC0415 - the caller's reference install
    if getattr(ref, "_b200_plugin", None) is not None:
        return ref._b200_plugin
    cls = backend_class(ref)
    bk = ref.backends
    orig_get = bk.get_backend
    names = tuple(bk.BACKEND_NAMES) + ("b200",)

    @functools.wraps(orig_get)
    def get_backend(name, **kwargs):
        if name == "b200":
            return cls(**kwargs)
        return orig_get(name, **kwargs)

    rebind = {(bk, "get_backend"): get_backend, (bk, "BACKEND_NAMES"): names}
    if fused:
        for mod, fname, pos, ours in _SOLVERS:
            orig = getattr(getattr(ref, mod), fname)
            rebind[(getattr(ref, mod), fname)] = _dispatch_backend(ref, orig, ours, pos)
        for mod, fname, ours in _FACTOR_SOLVES:
            orig = getattr(getattr(ref, mod), fname, None)
            if orig is not None:
                rebind[(getattr(ref, mod), fname)] = _dispatch_factor(ref, orig, ours)
    originals = {key[1]: getattr(*key) for key in rebind}
    # every loaded module of the package that imported one of these names gets the new binding
    for modname, mod in list(sys.modules.items()):
        if mod is None or not (modname == ref.__name__ or modname.startswith(ref.__name__ + ".")):
            continue
        for (_, attr), new in rebind.items():
            if getattr(mod, attr, None) is originals[attr]:
                setattr(mod, attr, new)
    ref._b200_plugin = cls
    ref._b200_rebind = {attr: new for (_, attr), new in rebind.items()}
    return cls


def rebind_module(ref, module) -> None:
    """Apply the plugin's bindings to a module that imported the reference's names before
    ``install`` ran (e.g. ``from densolve import cg_solve`` in a test file)."""
    new = getattr(ref, "_b200_rebind", {})
    for attr, fn in new.items():
        cur = getattr(module, attr, None)
        if cur is not None and cur is not fn and getattr(fn, "__wrapped__", None) is cur:
            setattr(module, attr, fn)


def _dispatch_backend(ref, orig, ours, pos):
    @functools.wraps(orig)
    def f(*args, **kwargs):
        be = args[pos] if len(args) > pos else kwargs.get("backend")
        if not _is_b200(be):
            return orig(*args, **kwargs)
        with _Translate(ref):
            return _convert_result(ref, ours(*args, **kwargs))
    return f


def _dispatch_factor(ref, orig, ours):
    @functools.wraps(orig)
    def f(fac, *args, **kwargs):
        mine = getattr(fac, "_b200", None)
        if mine is None:
            return orig(fac, *args, **kwargs)
        with _Translate(ref):
            return ours(mine, *args, **kwargs)
    return f
