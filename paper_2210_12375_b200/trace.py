"""NumPy dynamics callables -> device functors (the plugin surface).

The reference's dynamics are arbitrary NumPy callables ``f(t, y) -> (n, d)``
evaluated on the full batch (``pkg/src/batchode/stepper.py:19-20``).  The
persistent sm_100a integrator needs ``f`` inside the kernel, so a callable
is *traced*: it is called once with symbolic stand-ins for ``t`` (n,) and
``y`` (n, d) that record every NumPy operation (ufuncs, broadcasting,
indexing, ``np.where`` / ``np.stack`` / ...).  Every instance evaluates the
same expression, so the trace is one *row template* -- the expressions of a
single instance -- and the result is rendered as a CUDA functor
(``UserDyn``) with one scalar statement per operation, in NumPy's operation
order and rounding (``__dadd_rn`` / ``__dmul_rn`` / ... : NumPy never fuses).
Arrays the callable closes over become either literals (constant across
instances) or per-instance parameter columns (an axis of length n that
lines up with the instance axis, e.g. ``lam[:, None] * y``), which the
kernel loads once per instance.

What cannot be traced raises ``NotImplementedError`` -- there is no CPU
fallback: Python control flow on values (``if y[0, 0] > 1``), indexing
across instances, reductions over the batch, writing symbolic values into
a concrete NumPy array, or NumPy functions outside the supported set.
"""

import math

import numpy as np

__all__ = ["TraceError", "trace_dynamics", "TracedFunctor"]


class TraceError(NotImplementedError):
    pass


# ------------------------------------------------------------ expressions --
class Expr:
    __slots__ = ("op", "args", "kind", "value", "_h")

    def __init__(self, op, args=(), kind="f", value=None):
        self.op, self.args, self.kind, self.value = op, tuple(args), kind, value
        self._h = None


def _const(v):
    if isinstance(v, (bool, np.bool_)):
        return Expr("const", kind="b", value=bool(v))
    return Expr("const", value=float(v))


def _as_f(e):
    if e.kind == "b":  # NumPy promotes bool to 0.0 / 1.0
        return Expr("select", (e, _const(1.0), _const(0.0)))
    return e


# --------------------------------------------------------- symbolic arrays --
class Sym:
    """A batch array inside a traced dynamics call.  ``shape`` is the real
    NumPy shape (the instance axis has length n); ``E`` is the row template:
    an object array of the same shape with the instance axis of size 1."""

    __array_priority__ = 1000

    def __init__(self, tracer, shape, iaxis, E):
        self.tr, self.shape, self.iaxis, self.E = tracer, tuple(shape), iaxis, E

    # numpy protocol
    def __array_ufunc__(self, ufunc, method, *inputs, **kw):
        return self.tr.ufunc(ufunc, method, inputs, kw)

    def __array_function__(self, func, types, args, kwargs):
        return self.tr.function(func, args, kwargs)

    def __array__(self, *a, **k):
        raise TraceError("a traced dynamics value cannot be converted to a concrete NumPy array "
                         "(np.array / np.asarray / writing it into a NumPy buffer); build the "
                         "result with np.stack / np.empty_like + item assignment instead")

    def __bool__(self):
        raise TraceError("Python control flow on state values cannot run inside the device "
                         "solver; use np.where")

    def __float__(self):
        raise TraceError("a traced dynamics value has no concrete float value")

    __int__ = __index__ = __float__

    def __len__(self):
        return self.shape[0]

    def __iter__(self):
        raise TraceError("iterating over a traced batch array is not supported")

    # attributes numpy code commonly touches
    @property
    def ndim(self):
        return len(self.shape)

    @property
    def size(self):
        return int(np.prod(self.shape))

    @property
    def dtype(self):
        return np.dtype(bool) if self.E.size and all(e.kind == "b" for e in self.E.flat) \
            else np.dtype(np.float64)

    @property
    def T(self):
        return self.transpose()

    def transpose(self, *axes):
        axes = axes[0] if len(axes) == 1 and isinstance(axes[0], (tuple, list)) else axes
        axes = tuple(axes) if axes else tuple(range(self.ndim))[::-1]
        return Sym(self.tr, tuple(self.shape[a] for a in axes), axes.index(self.iaxis),
                   self.E.transpose(axes))

    def copy(self, *a, **k):
        return Sym(self.tr, self.shape, self.iaxis, self.E.copy())

    def astype(self, dtype, *a, **k):
        dt = np.dtype(dtype)
        if dt == np.dtype(bool):
            return self.tr.ufunc(np.not_equal, "__call__", (self, 0.0), {})
        if dt.kind != "f":
            raise TraceError(f"cast to {dt} is not supported in traced dynamics")
        return Sym(self.tr, self.shape, self.iaxis, np.vectorize(_as_f, otypes=[object])(self.E)
                   if self.E.size else self.E.copy())

    def reshape(self, *shape):
        shape = shape[0] if len(shape) == 1 and isinstance(shape[0], (tuple, list)) else shape
        return self.tr.reshape(self, tuple(shape))

    def sum(self, axis=None, keepdims=False, **k):
        return self.tr.reduce_sum(self, axis, keepdims)

    def mean(self, axis=None, keepdims=False, **k):
        return self.tr.mean(self, axis, keepdims)

    def dot(self, other):
        return np.dot(self, other)

    def __getitem__(self, idx):
        return self.tr.getitem(self, idx)

    def __setitem__(self, idx, value):
        self.tr.setitem(self, idx, value)

    # operators -> ufuncs (so Python scalars on either side work)
    def _u(f, swap=False):
        if swap:
            return lambda s, o: f(o, s)
        return lambda s, o: f(s, o)

    __add__, __radd__ = _u(np.add), _u(np.add, True)
    __sub__, __rsub__ = _u(np.subtract), _u(np.subtract, True)
    __mul__, __rmul__ = _u(np.multiply), _u(np.multiply, True)
    __truediv__, __rtruediv__ = _u(np.true_divide), _u(np.true_divide, True)
    __matmul__, __rmatmul__ = _u(np.matmul), _u(np.matmul, True)
    __lt__, __le__ = _u(np.less), _u(np.less_equal)
    __gt__, __ge__ = _u(np.greater), _u(np.greater_equal)
    __eq__, __ne__ = _u(np.equal), _u(np.not_equal)
    __and__, __or__ = _u(np.logical_and), _u(np.logical_or)
    __rpow__ = _u(np.power, True)
    __hash__ = None

    def __pow__(self, e):
        # ndarray ** python scalar takes NumPy's fast_scalar_power short cuts
        if np.ndim(e) == 0 and not isinstance(e, Sym):
            ev = float(e)
            if ev == 2.0:
                return np.square(self)
            if ev == 0.5:
                return np.sqrt(self)
            if ev == -1.0:
                return np.reciprocal(self)
            if ev == 1.0:
                return self.copy()
            if ev == 0.0:
                return self.tr.full_like(self, 1.0)
        return np.power(self, e)

    def __neg__(self):
        return np.negative(self)

    def __pos__(self):
        return self.copy()

    def __abs__(self):
        return np.absolute(self)

    def __invert__(self):
        return np.logical_not(self)

    del _u


# unary / binary ufuncs -> expression ops
_UNARY = {np.negative: "neg", np.positive: "pos", np.absolute: "abs", np.fabs: "abs",
          np.sqrt: "sqrt", np.square: "square", np.reciprocal: "recip", np.exp: "exp",
          np.expm1: "expm1", np.exp2: "exp2", np.log: "log", np.log1p: "log1p",
          np.log2: "log2", np.log10: "log10", np.sin: "sin", np.cos: "cos", np.tan: "tan",
          np.arcsin: "asin", np.arccos: "acos", np.arctan: "atan", np.sinh: "sinh",
          np.cosh: "cosh", np.tanh: "tanh", np.arcsinh: "asinh", np.arccosh: "acosh",
          np.arctanh: "atanh", np.cbrt: "cbrt", np.floor: "floor", np.ceil: "ceil",
          np.rint: "rint", np.trunc: "trunc", np.sign: "sign", np.isfinite: "isfinite",
          np.isnan: "isnan", np.isinf: "isinf", np.logical_not: "not", np.signbit: "signbit"}
_BINARY = {np.add: "add", np.subtract: "sub", np.multiply: "mul", np.true_divide: "div",
           np.power: "pow", np.maximum: "max", np.minimum: "min", np.fmax: "fmax",
           np.fmin: "fmin", np.arctan2: "atan2", np.hypot: "hypot", np.copysign: "copysign",
           np.fmod: "fmod", np.greater: "gt", np.greater_equal: "ge", np.less: "lt",
           np.less_equal: "le", np.equal: "eq", np.not_equal: "ne",
           np.logical_and: "and", np.logical_or: "or", np.logical_xor: "xor"}
_BOOL_OUT = {"isfinite", "isnan", "isinf", "not", "signbit", "gt", "ge", "lt", "le", "eq", "ne",
             "and", "or", "xor"}
_BOOL_IN = {"not", "and", "or", "xor"}


class Tracer:
    def __init__(self, n, d):
        self.n, self.d = n, d
        self.params = []      # per-instance columns (length-n float arrays)
        self._pkeys = {}

    # ---------------------------------------------------------- operands --
    def sym(self, shape, iaxis, E):
        return Sym(self, shape, iaxis, E)

    def param(self, col):
        """A per-instance column (1-D, length n) -> Expr('param', k)."""
        col = np.asarray(col)
        ai = col.__array_interface__
        key = (ai["data"][0], col.strides, col.dtype.str, col.shape)
        k = self._pkeys.get(key)
        if k is None:
            k = len(self.params)
            self.params.append(np.asarray(col, dtype=np.float64))
            self._pkeys[key] = k
        return Expr("param", value=k)

    def template(self, x, rshape, raxis):
        """Row template of operand x broadcast to the real shape rshape whose
        instance axis is raxis (None: no instance axis)."""
        if isinstance(x, Sym):
            off = len(rshape) - x.ndim
            tshape = list(rshape)
            if raxis is not None:
                tshape[raxis] = 1
            src = x.E.reshape((1,) * off + x.E.shape)
            return np.broadcast_to(src, tshape)
        a = np.asarray(x)
        if a.dtype == object:
            raise TraceError("object arrays cannot enter traced dynamics")
        if a.dtype.kind not in "biuf":
            raise TraceError(f"dtype {a.dtype} cannot enter traced dynamics")
        off = len(rshape) - a.ndim
        full = np.broadcast_to(a, rshape)
        tshape = list(rshape)
        if raxis is not None:
            tshape[raxis] = 1
        out = np.empty(tshape, dtype=object)
        per_inst = (raxis is not None and raxis >= off and a.shape[raxis - off] == self.n
                    and self.n > 1)
        for pos in np.ndindex(*tshape):
            if per_inst:
                idx = list(pos)
                idx[raxis] = slice(None)
                out[pos] = self.param(full[tuple(idx)])
            else:
                out[pos] = _const(full[pos] if a.dtype.kind == "b" else float(full[pos]))
        return out

    def result_frame(self, operands):
        """numpy broadcasting of the real shapes -> (shape, instance axis)."""
        shapes = [o.shape if isinstance(o, Sym) else np.shape(o) for o in operands]
        try:
            rshape = np.broadcast_shapes(*shapes)
        except ValueError as e:
            raise ValueError(str(e)) from None
        raxis = None
        for o in operands:
            if isinstance(o, Sym):
                ax = len(rshape) - o.ndim + o.iaxis
                if raxis is None:
                    raxis = ax
                elif raxis != ax:
                    raise TraceError("an operation mixes different instances (misaligned "
                                     "instance axes)")
        return rshape, raxis

    # ------------------------------------------------------------ ufuncs --
    def ufunc(self, uf, method, inputs, kw):
        if method != "__call__":
            raise TraceError(f"np.{uf.__name__}.{method} is not supported in traced dynamics")
        if kw.get("out") is not None or kw.get("where", True) is not True:
            raise TraceError("ufunc out= / where= are not supported in traced dynamics")
        if uf is np.matmul:
            return self.matmul(*inputs)
        rshape, raxis = self.result_frame(inputs)
        ts = [self.template(x, rshape, raxis) for x in inputs]
        if uf in _UNARY and len(inputs) == 1:
            op = _UNARY[uf]
            fn = lambda a: self.node(op, (a,))  # noqa: E731
        elif uf in _BINARY and len(inputs) == 2:
            op = _BINARY[uf]
            fn = lambda a, b: self.node(op, (a, b))  # noqa: E731
        else:
            raise TraceError(f"np.{uf.__name__} is not supported in traced dynamics")
        out = np.empty(ts[0].shape, dtype=object)
        for pos in np.ndindex(*out.shape):
            out[pos] = fn(*(t[pos] for t in ts))
        if raxis is None:  # only constants: fold to a concrete result
            return self.fold(out)
        return Sym(self, rshape, raxis, out)

    def fold(self, E):
        vals = np.empty(E.shape, dtype=object)
        for pos in np.ndindex(*E.shape):
            e = E[pos]
            if e.op != "const":
                raise TraceError("internal: constant folding of a non-constant")
            vals[pos] = e.value
        return np.array(vals.tolist(), dtype=bool if E.size and E.flat[0].kind == "b" else float)

    def node(self, op, args):
        if op in _BOOL_IN:
            args = tuple(a if a.kind == "b" else Expr("ne", (a, _const(0.0)), kind="b")
                         for a in args)
        else:
            args = tuple(_as_f(a) for a in args)
        if all(a.op == "const" for a in args):  # fold with NumPy itself
            vals = [np.bool_(a.value) if a.kind == "b" else np.float64(a.value) for a in args]
            uf = {v: k for k, v in {**_UNARY, **_BINARY}.items()}[op] if op != "square" \
                else np.square
            with np.errstate(all="ignore"):
                r = uf(*vals)
            return _const(bool(r) if op in _BOOL_OUT else float(r))
        return Expr(op, args, kind="b" if op in _BOOL_OUT else "f")

    # ---------------------------------------------------------- indexing --
    def _norm_index(self, s, idx):
        if not isinstance(idx, tuple):
            idx = (idx,)
        n_real = sum(1 for i in idx if i is not None and i is not Ellipsis)
        out, used = [], 0
        for i in idx:
            if i is Ellipsis:
                out.extend([slice(None)] * (s.ndim - n_real))
                used += s.ndim - n_real
            else:
                out.append(i)
                if i is not None:
                    used += 1
        out.extend([slice(None)] * (s.ndim - used))
        return out

    def _check_instance_component(self, s, comps):
        ax = 0
        for c in comps:
            if c is None:
                continue
            if ax == s.iaxis:
                if not (isinstance(c, slice) and c == slice(None) or
                        (isinstance(c, slice) and slice(*c.indices(self.n)) == slice(0, self.n, 1))):
                    raise TraceError("indexing along the instance (batch) axis is not supported "
                                     "in traced dynamics")
            ax += 1

    def getitem(self, s, idx):
        comps = self._norm_index(s, idx)
        self._check_instance_component(s, comps)
        tcomps = []
        ax = 0
        for c in comps:
            if c is None:
                tcomps.append(None)
                continue
            tcomps.append(slice(None) if ax == s.iaxis else c)
            ax += 1
        # instance-axis position after indexing: index a small probe whose
        # instance axis has length 2 and find the axis it lands on
        pshape = list(s.shape)
        pshape[s.iaxis] = 2
        probe = np.broadcast_to(np.arange(2).reshape([2 if a == s.iaxis else 1
                                                      for a in range(s.ndim)]), pshape)
        pr = probe[tuple(tcomps)]
        axes = [a for a in range(pr.ndim) if pr.shape[a] == 2 and
                np.any(np.take(pr, 0, axis=a) != np.take(pr, 1, axis=a))]
        if len(axes) != 1:
            raise TraceError("unsupported indexing of a traced batch array")
        E = s.E[tuple(tcomps)]
        rshape = np.broadcast_to(np.zeros((), bool), s.shape)[tuple(comps)].shape
        return Sym(self, rshape, axes[0], E)

    def setitem(self, s, idx, value):
        comps = self._norm_index(s, idx)
        self._check_instance_component(s, comps)
        tcomps = []
        ax = 0
        for c in comps:
            if c is None:
                tcomps.append(None)
                continue
            tcomps.append(slice(None) if ax == s.iaxis else c)
            ax += 1
        view_shape = np.broadcast_to(np.zeros((), bool), s.shape)[tuple(comps)].shape
        tgt = s.E[tuple(tcomps)]
        # instance axis of the target view, as in getitem
        probe_shape = list(s.shape)
        probe_shape[s.iaxis] = 2
        probe = np.broadcast_to(np.arange(2).reshape([2 if a == s.iaxis else 1
                                                      for a in range(s.ndim)]), probe_shape)
        pr = probe[tuple(tcomps)]
        axes = [a for a in range(pr.ndim) if pr.shape[a] == 2 and
                np.any(np.take(pr, 0, axis=a) != np.take(pr, 1, axis=a))]
        raxis = axes[0] if len(axes) == 1 else None
        if isinstance(value, Sym):
            vax = len(view_shape) - value.ndim + value.iaxis
            if vax != raxis:
                raise TraceError("assignment mixes different instances")
        vt = self.template(value, view_shape, raxis)
        if vt.shape != tgt.shape:
            vt = np.broadcast_to(vt, tgt.shape)
        s.E[tuple(tcomps)] = vt

    # ----------------------------------------------------------- helpers --
    def full_like(self, s, v):
        E = np.empty(s.E.shape, dtype=object)
        for pos in np.ndindex(*E.shape):
            E[pos] = _const(v)
        return Sym(self, s.shape, s.iaxis, E)

    def reshape(self, s, shape):
        shape = tuple(int(x) for x in shape)
        if -1 in shape:
            k = shape.index(-1)
            rest = int(np.prod([x for x in shape if x != -1]))
            shape = shape[:k] + (int(np.prod(s.shape)) // rest,) + shape[k + 1:]
        # only reshapes that keep the leading instance axis and regroup the rest
        if s.iaxis != 0 or shape[0] != s.shape[0]:
            raise TraceError("reshape must keep the leading instance axis")
        return Sym(self, shape, 0, s.E.reshape((1,) + shape[1:]))

    def _axis(self, s, axis):
        if axis is None:
            raise TraceError("reductions over the instance (batch) axis are not supported")
        axis = axis + s.ndim if axis < 0 else axis
        if axis == s.iaxis:
            raise TraceError("reductions over the instance (batch) axis are not supported")
        return axis

    def reduce_sum(self, s, axis, keepdims):
        if not isinstance(s, Sym):
            return np.sum(s, axis=axis, keepdims=keepdims)
        axis = self._axis(s, axis)
        E = np.moveaxis(s.E, axis, -1)
        out = np.empty(E.shape[:-1], dtype=object)
        for pos in np.ndindex(*out.shape):
            out[pos] = self._pairwise([_as_f(e) for e in E[pos]])
        shape = s.shape[:axis] + s.shape[axis + 1:]
        iaxis = s.iaxis - (1 if s.iaxis > axis else 0)
        r = Sym(self, shape, iaxis, out)
        if keepdims:
            r = r[(slice(None),) * axis + (None,)]
        return r

    def _pairwise(self, xs):
        # NumPy's pairwise summation (umath loops_utils pairwise_sum): below 8
        # terms a running sum seeded with 0.0, up to 128 eight strided
        # accumulators, beyond that a recursive halving at a multiple of 8 --
        # the order bode_device.cuh pairwise_sum reproduces for error_norm
        n = len(xs)
        if n < 8:
            r = _const(0.0)
            for x in xs:
                r = self.node("add", (r, x))
            return r
        if n <= 128:
            r = list(xs[:8])
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] = self.node("add", (r[j], xs[i + j]))
                i += 8
            res = self.node("add", (self.node("add", (self.node("add", (r[0], r[1])),
                                                      self.node("add", (r[2], r[3])))),
                                    self.node("add", (self.node("add", (r[4], r[5])),
                                                      self.node("add", (r[6], r[7]))))))
            for k in range(n - (n % 8), n):
                res = self.node("add", (res, xs[k]))
            return res
        h = n // 2
        h -= h % 8
        return self.node("add", (self._pairwise(xs[:h]), self._pairwise(xs[h:])))

    def mean(self, s, axis, keepdims):
        r = self.reduce_sum(s, axis, keepdims)
        cnt = s.shape[self._axis(s, axis)]
        return np.true_divide(r, float(cnt))

    def matmul(self, a, b):
        if isinstance(a, Sym) and isinstance(b, Sym):
            raise TraceError("products of two traced batch arrays over the state axis are "
                             "not supported (write them elementwise)")
        if isinstance(a, Sym):
            B = np.asarray(b, dtype=float)
            if a.ndim != 2 or a.iaxis != 0 or B.ndim not in (1, 2) or B.shape[0] != a.shape[1]:
                raise TraceError("matmul: (n, d) @ (d, k) or (d,) with a constant right operand")
            Bm = B if B.ndim == 2 else B[:, None]
            out = np.empty((1, Bm.shape[1]), dtype=object)
            for k in range(Bm.shape[1]):
                acc = None
                for j in range(Bm.shape[0]):
                    term = self.node("mul", (a.E[0, j], _const(Bm[j, k])))
                    acc = term if acc is None else self.node("add", (acc, term))
                out[0, k] = acc
            if B.ndim == 1:
                return Sym(self, (a.shape[0],), 0, out[:, 0])
            return Sym(self, (a.shape[0], Bm.shape[1]), 0, out)
        if isinstance(b, Sym):
            A = np.asarray(a, dtype=float)
            if b.ndim != 2 or b.iaxis != 1 or A.ndim != 2 or A.shape[1] != b.shape[0]:
                raise TraceError("matmul: (k, d) @ (d, n) with a constant left operand")
            out = np.empty((A.shape[0], 1), dtype=object)
            for k in range(A.shape[0]):
                acc = None
                for j in range(A.shape[1]):
                    term = self.node("mul", (_const(A[k, j]), b.E[j, 0]))
                    acc = term if acc is None else self.node("add", (acc, term))
                out[k, 0] = acc
            return Sym(self, (A.shape[0], b.shape[1]), 1, out)
        return np.matmul(a, b)

    # ----------------------------------------------------- array functions --
    def function(self, func, args, kwargs):
        name = func.__name__
        if name in ("zeros_like", "ones_like", "empty_like", "full_like"):
            s = args[0]
            if kwargs.get("shape") is not None:
                raise TraceError(f"np.{name}(shape=...) is not supported")
            v = {"zeros_like": 0.0, "ones_like": 1.0, "empty_like": 0.0}.get(name)
            if name == "full_like":
                v = args[1] if len(args) > 1 else kwargs["fill_value"]
                if isinstance(v, Sym):
                    raise TraceError("np.full_like with a traced fill value")
            dt = kwargs.get("dtype", args[2] if name == "full_like" and len(args) > 2 else None)
            if dt is not None and np.dtype(dt) == np.dtype(bool):
                v = bool(v)
            return self.full_like(s, v)
        if name == "where":
            if len(args) + len(kwargs) != 3:
                raise TraceError("np.where(cond) (index form) is not supported")
            c, a, b = args
            rshape, raxis = self.result_frame([c, a, b])
            tc, ta, tb = (self.template(x, rshape, raxis) for x in (c, a, b))
            out = np.empty(tc.shape, dtype=object)
            for pos in np.ndindex(*out.shape):
                cond = tc[pos] if tc[pos].kind == "b" else Expr("ne", (tc[pos], _const(0.0)),
                                                                kind="b")
                x, y = ta[pos], tb[pos]
                kind = "b" if x.kind == "b" and y.kind == "b" else "f"
                if kind == "f":
                    x, y = _as_f(x), _as_f(y)
                if cond.op == "const":
                    out[pos] = x if cond.value else y
                else:
                    out[pos] = Expr("select", (cond, x, y), kind=kind)
            if raxis is None:
                return self.fold(out)
            return Sym(self, rshape, raxis, out)
        if name in ("stack", "concatenate", "column_stack", "hstack", "vstack"):
            seq = list(args[0])
            axis = kwargs.get("axis", args[1] if len(args) > 1 else 0)
            if name == "column_stack":
                seq = [s[:, None] if (isinstance(s, Sym) and s.ndim == 1) or np.ndim(s) == 1
                       else s for s in seq]
                name, axis = "concatenate", 1
            elif name == "hstack":
                name, axis = "concatenate", (0 if all(np.ndim(s) == 1 for s in seq) else 1)
            elif name == "vstack":
                seq = [s[None, :] if ((isinstance(s, Sym) and s.ndim == 1) or np.ndim(s) == 1)
                       else s for s in seq]
                name, axis = "concatenate", 0
            return self.join(seq, axis, stack=name == "stack")
        if name == "clip":
            a = args[0]
            lo = kwargs.get("a_min", kwargs.get("min", args[1] if len(args) > 1 else None))
            hi = kwargs.get("a_max", kwargs.get("max", args[2] if len(args) > 2 else None))
            r = a
            if lo is not None:
                r = np.maximum(r, lo)
            if hi is not None:
                r = np.minimum(r, hi)
            return r
        if name == "sum":
            return self.reduce_sum(args[0], kwargs.get("axis", args[1] if len(args) > 1 else None),
                                   kwargs.get("keepdims", False))
        if name == "mean":
            return self.mean(args[0], kwargs.get("axis", args[1] if len(args) > 1 else None),
                             kwargs.get("keepdims", False))
        if name in ("dot", "inner") and name == "dot":
            return self.matmul(*args)
        if name == "transpose":
            axes = kwargs.get("axes", args[1] if len(args) > 1 else None)
            return args[0].transpose(*(() if axes is None else (tuple(axes),)))
        if name in ("copy", "asarray", "asanyarray", "array") and isinstance(args[0], Sym):
            dt = kwargs.get("dtype", args[1] if len(args) > 1 else None)
            return args[0].astype(dt) if dt is not None else args[0].copy()
        if name == "expand_dims":
            s, ax = args[0], kwargs.get("axis", args[1] if len(args) > 1 else None)
            ax = ax + s.ndim + 1 if ax < 0 else ax
            return s[(slice(None),) * ax + (None,)]
        if name == "broadcast_to":
            s, shape = args[0], tuple(kwargs.get("shape", args[1] if len(args) > 1 else ()))
            rshape, raxis = self.result_frame([s, np.broadcast_to(0.0, shape)])
            if rshape != shape:
                raise ValueError("operands could not be broadcast")
            return Sym(self, rshape, raxis, np.array(self.template(s, rshape, raxis)))
        if name == "reshape":
            return self.reshape(args[0], kwargs.get("newshape", kwargs.get("shape", args[1])))
        if name in ("shape", "ndim", "size"):
            return getattr(args[0], name)
        raise TraceError(f"np.{name} is not supported in traced dynamics")

    def join(self, seq, axis, stack):
        syms = [s for s in seq if isinstance(s, Sym)]
        if not syms:
            return (np.stack if stack else np.concatenate)(seq, axis=axis)
        if stack:
            seq = [s[(slice(None),) * (axis if axis >= 0 else s.ndim + 1 + axis) + (None,)]
                   if isinstance(s, Sym) else np.expand_dims(np.asarray(s), axis) for s in seq]
            axis = axis if axis >= 0 else seq[0].ndim + axis
            syms = [s for s in seq if isinstance(s, Sym)]
        nd = max((s.ndim if isinstance(s, Sym) else np.ndim(s)) for s in seq)
        axis = axis + nd if axis < 0 else axis
        ref = syms[0]
        iax = ref.iaxis
        if iax == axis:
            raise TraceError("concatenating along the instance (batch) axis is not supported")
        parts, shapes = [], []
        for s in seq:
            shp = list(s.shape if isinstance(s, Sym) else np.shape(s))
            if len(shp) != nd:
                raise ValueError("all the input arrays must have same number of dimensions")
            full = list(ref.shape)
            full[axis] = shp[axis]
            if isinstance(s, Sym) and s.iaxis != iax:
                raise TraceError("joining arrays with different instance axes")
            t = self.template(s, tuple(full), iax)
            parts.append(t)
            shapes.append(shp[axis])
        E = np.concatenate(parts, axis=axis)
        shape = list(ref.shape)
        shape[axis] = sum(shapes)
        return Sym(self, tuple(shape), iax, E)


# ------------------------------------------------------------ code render --
_FN1 = {"exp": "exp", "expm1": "expm1", "exp2": "exp2", "log": "log", "log1p": "log1p",
        "log2": "log2", "log10": "log10", "sin": "sin", "cos": "cos", "tan": "tan",
        "asin": "asin", "acos": "acos", "atan": "atan", "sinh": "sinh", "cosh": "cosh",
        "tanh": "tanh", "asinh": "asinh", "acosh": "acosh", "atanh": "atanh", "cbrt": "cbrt",
        "floor": "floor", "ceil": "ceil", "rint": "rint", "trunc": "trunc", "abs": "fabs"}
_FN2 = {"fmax": "fmax", "fmin": "fmin", "atan2": "atan2", "hypot": "hypot",
        "copysign": "copysign", "fmod": "fmod"}
_CMP = {"gt": ">", "ge": ">=", "lt": "<", "le": "<=", "eq": "==", "ne": "!="}


def _lit(v, kind):
    if kind == "b":
        return "true" if v else "false"
    if math.isnan(v):
        return "__longlong_as_double(0x7ff8000000000000LL)"
    if math.isinf(v):
        return ("__longlong_as_double(0x7ff0000000000000LL)" if v > 0
                else "__longlong_as_double(0xfff0000000000000LL)")
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    return f"{v.hex()} /* {v!r} */"


class TracedFunctor:
    """A traced dynamics: CUDA source of ``bode::UserDyn<O>``, the
    per-instance parameter columns it reads (n, P) and a structural key."""

    def __init__(self, source, params, d, key):
        self.source, self.params, self.d, self.key = source, params, d, key


def _render(out_exprs, d, n_params):
    lines, memo = [], {}
    counter = [0]

    def emit(e):
        k = id(e)
        if k in memo:
            return memo[k]
        op = e.op
        if op == "const":
            r = _lit(e.value, e.kind)
            memo[k] = r
            return r
        if op == "y":
            r = f"y[{e.value}]"
            memo[k] = r
            return r
        if op == "t":
            memo[k] = "t"
            return "t"
        if op == "param":
            r = f"p[{e.value}]"
            memo[k] = r
            return r
        a = [emit(x) for x in e.args]
        if op == "add":
            x = f"__dadd_rn({a[0]}, {a[1]})"
        elif op == "sub":
            x = f"__dsub_rn({a[0]}, {a[1]})"
        elif op == "mul":
            x = f"__dmul_rn({a[0]}, {a[1]})"
        elif op == "div":
            x = f"__ddiv_rn({a[0]}, {a[1]})"
        elif op == "neg":
            x = f"(-{a[0]})"
        elif op == "pos":
            x = a[0]
        elif op == "sqrt":
            x = f"__dsqrt_rn({a[0]})"
        elif op == "square":
            x = f"__dmul_rn({a[0]}, {a[0]})"
        elif op == "recip":
            x = f"__ddiv_rn(1.0, {a[0]})"
        elif op == "pow":
            x = f"bode::user_pow({a[0]}, {a[1]})"
        elif op == "max":
            x = f"bode::np_max({a[0]}, {a[1]})"
        elif op == "min":
            x = f"bode::np_min({a[0]}, {a[1]})"
        elif op == "sign":
            x = f"bode::user_sign({a[0]})"
        elif op in _FN1:
            x = f"{_FN1[op]}({a[0]})"
        elif op in _FN2:
            x = f"{_FN2[op]}({a[0]}, {a[1]})"
        elif op in _CMP:
            x = f"({a[0]} {_CMP[op]} {a[1]})"
        elif op == "and":
            x = f"({a[0]} && {a[1]})"
        elif op == "or":
            x = f"({a[0]} || {a[1]})"
        elif op == "xor":
            x = f"({a[0]} != {a[1]})"
        elif op == "not":
            x = f"(!{a[0]})"
        elif op == "isfinite":
            x = f"isfinite({a[0]})"
        elif op == "isnan":
            x = f"isnan({a[0]})"
        elif op == "isinf":
            x = f"isinf({a[0]})"
        elif op == "signbit":
            x = f"signbit({a[0]})"
        elif op == "select":
            x = f"({a[0]} ? {a[1]} : {a[2]})"
        else:
            raise TraceError(f"internal: no rendering for {op}")
        v = f"v{counter[0]}"
        counter[0] += 1
        ctype = "bool" if e.kind == "b" else "double"
        lines.append(f"    const {ctype} {v} = {x};")
        memo[k] = v
        return v

    outs = [emit(_as_f(e)) for e in out_exprs]
    body = "\n".join(lines)
    assigns = "\n".join(f"    f[{j}] = {o};" for j, o in enumerate(outs))
    if n_params > 24:  # wide parameter rows stay in global memory (L1-cached loads)
        pdecl = "const double* p;"
        load = "    p = P.inst + i * NP;"
    else:
        pdecl = f"double p[{max(n_params, 1)}];"
        load = ("    for (int k = 0; k < NP; k++) p[k] = P.inst[i * NP + k];" if n_params
                else "    (void)P; (void)i;")
    return f"""namespace bode {{
// NumPy's array ** array (libm pow; correctly rounded here, bode_pow.cuh)
__device__ __forceinline__ double user_pow(double x, double e) {{ return np_scalar_pow(x, e); }}
__device__ __forceinline__ double user_sign(double x) {{
  return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : (x == 0.0 ? 0.0 : x));
}}
template <class O>
struct UserDyn {{  // traced from the caller's NumPy dynamics (trace.py)
  static constexpr int D = {d};
  static constexpr int NP = {n_params};
  {pdecl}
  __device__ __forceinline__ void load(const DynParams& P, int64_t i) {{
{load}
  }}
  __device__ __forceinline__ void operator()(double t, const double* y, double* f) const {{
    (void)t;
{body}
{assigns}
  }}
}};
}}  // namespace bode
"""


def trace_dynamics(f, n: int, d: int) -> TracedFunctor:
    """Trace ``f(t, y)`` for a batch of n instances of width d."""
    tr = Tracer(n, d)
    tE = np.empty((1,), dtype=object)
    tE[0] = Expr("t")
    yE = np.empty((1, d), dtype=object)
    for j in range(d):
        yE[0, j] = Expr("y", value=j)
    t = Sym(tr, (n,), 0, tE)
    y = Sym(tr, (n, d), 0, yE)
    try:
        with np.errstate(all="ignore"):
            r = f(t, y)
    except TraceError:
        raise
    except (TypeError, AttributeError) as e:
        raise TraceError(f"dynamics {getattr(f, '__name__', f)!r} could not be traced for the "
                         f"device solver: {e}") from e
    if isinstance(r, (list, tuple)):
        r = np.stack(r, axis=-1) if any(isinstance(x, Sym) for x in r) else np.asarray(r)
    if isinstance(r, Sym):
        if r.shape != (n, d):
            if r.shape == (n,) and d == 1:
                r = r[:, None]
            else:
                raise ValueError(f"dynamics returned shape {r.shape}, expected {(n, d)}")
        if r.iaxis != 0:
            raise TraceError("dynamics result's leading axis is not the instance axis")
        outs = list(r.E[0])
    else:
        a = np.broadcast_to(np.asarray(r, dtype=float), (n, d))
        outs = list(tr.template(a, (n, d), 0)[0])
    src = _render(outs, d, len(tr.params))
    params = np.stack(tr.params, axis=1) if tr.params else None
    return TracedFunctor(src, params, d, src)
