"""Route the reference's own code onto the device operators (the drop-in at SURVEY.md §8(b)).

The reference (``factorla``) has no FFI layer; its hot path sits behind three Python
surfaces: the ``rewrite`` operator functions, the ML drivers' polymorphic helpers
(ml.py:101-180, which dispatch on ``isinstance(m, NormalizedMatrix)`` of the *reference's*
class and call ``rewrite.*``), and the cost model's op registry (costmodel.py:161-172).
``route_reference_drivers`` patches the drivers' helpers so that a matrix built with
``paper_1612_07448_b200.build_*`` runs every ``ml.logistic_gd / linreg_gd / linreg_normal /
kmeans / gnmf`` operator call on the device, while the reference's own matrices keep
their CPU path:

* ``ml._is_nm``      (ml.py:101-102) accepts both classes;
* ``ml.rewrite``     (used by ml.py:105-152) becomes a dispatcher: the device operators for
                     device matrices, the reference's ``rewrite`` for its own;
* ``ml._take_rows``  (ml.py:155-168) gathers seed rows on the device (the reference calls
                     ``ndarray.take`` on the blocks);
* ``ml._min_value``  (ml.py:171-180) reduces the device factors.

``register_cost_model_ops`` puts the device operators into ``costmodel._FACTORIZED_OPS``.
Both return an ``undo()`` callable restoring the reference's attributes.
"""

from . import ml as _fbml
from . import normmat as _fbnm
from . import rewrite as _fbrw

__all__ = ["route_reference_drivers", "register_cost_model_ops"]


def _is_device(m):
    return isinstance(m, _fbnm.NormalizedMatrix)


class _RewriteDispatch:
    """Stands in for the ``factorla.rewrite`` module inside ``factorla.ml``."""

    def __init__(self, ref_rewrite):
        self._ref = ref_rewrite

    def __getattr__(self, name):
        ref_fn = getattr(self._ref, name)
        dev_fn = getattr(_fbrw, name, None)

        def call(*args, **kwargs):
            # the normalized operand is the first positional argument of every operator the
            # drivers call (lmm, scalar_op, scalar_fn, row_sums, sum_all, crossprod,
            # gram_transposed); rmm takes it second
            nm = args[1] if name == "rmm" and len(args) > 1 else (args[0] if args else None)
            if dev_fn is not None and _is_device(nm):
                return dev_fn(*args, **kwargs)
            return ref_fn(*args, **kwargs)

        return call


def route_reference_drivers(factorla):
    """Patch ``factorla.ml`` so its drivers run device matrices on the sm_100a operators."""
    ml = factorla.ml
    saved = {k: getattr(ml, k) for k in ("_is_nm", "rewrite", "_take_rows", "_min_value")}
    ref_is_nm, ref_take, ref_min = saved["_is_nm"], saved["_take_rows"], saved["_min_value"]

    def _is_nm(m):
        return _is_device(m) or ref_is_nm(m)

    def _take_rows(m, idx):
        if _is_device(m):
            if m.transposed:
                raise factorla.ShapeError("row sampling expects an untransposed matrix")
            return _fbml._take_rows(m, idx).cpu().numpy()
        return ref_take(m, idx)

    def _min_value(m):
        return _fbml._min_value(m) if _is_device(m) else ref_min(m)

    ml._is_nm = _is_nm
    ml.rewrite = _RewriteDispatch(saved["rewrite"])
    ml._take_rows = _take_rows
    ml._min_value = _min_value

    def undo():
        for k, v in saved.items():
            setattr(ml, k, v)

    return undo


def register_cost_model_ops(factorla):
    """Device operators in the cost model's registry (costmodel.py:161-172): the factorized
    plan of ``auto_dispatch`` then runs on the device for device matrices."""
    cm = factorla.costmodel
    reg = cm._FACTORIZED_OPS
    saved = dict(reg)

    def pick(name, dev):
        ref = saved[name]

        def op(nm, counter, *a, **k):
            return dev(nm, counter, *a, **k) if _is_device(nm) else ref(nm, counter, *a, **k)

        return op

    dev_ops = {  # same ids and keyword arguments as the reference's registry
        "scalar_op": lambda nm, c, x=1.0, op="mul": _fbrw.scalar_op(nm, x, op, c),
        "scalar_fn": lambda nm, c, f=None: _fbrw.scalar_fn(nm, f, c),
        "rowsums": lambda nm, c: _fbrw.row_sums(nm, c),
        "colsums": lambda nm, c: _fbrw.col_sums(nm, c),
        "sum": lambda nm, c: _fbrw.sum_all(nm, c),
        "lmm": lambda nm, c, x=None: _fbrw.lmm(nm, x, c),
        "rmm": lambda nm, c, x=None: _fbrw.rmm(x, nm, c),
        "crossprod": lambda nm, c, method="efficient": _fbrw.crossprod(nm, method, c),
        "gram_transposed": lambda nm, c: _fbrw.gram_transposed(nm, c),
        "ginv": lambda nm, c: _fbrw.ginv(nm, c),
    }
    for name, dev in dev_ops.items():
        if name in reg:
            reg[name] = pick(name, dev)

    def undo():
        reg.clear()
        reg.update(saved)

    return undo
