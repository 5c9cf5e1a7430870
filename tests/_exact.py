"""Exact rational primal definitions + forward-mode dual numbers (test-only).

These are the *primal* definitions of the paper's combinators, written out in
plain Python over ``fractions.Fraction`` so that every value is exact:

  scan            P:1136-1137  [a0, a0(.)a1, ..., a0(.)...(.)a_{n-1}]
  reduce          P:975-977    a0 (.) a1 (.) ... (.) a_{n-1}
  reduce_by_index P:1102-1105  hs = replicate m e; hs[inds[i]] (.)= as[i]
  scatter         P:1241-1244  ys = xs with ys[is[j]] = vs[j]

Forward mode is the dual-number reading of Eq. 2:
each scalar carries (value, tangent).  Mapping the jvp over the standard basis
 recovers Jacobian columns, so  abar_k = <ybar, J e_k>  is computed
by a route entirely different from the oracle's reverse loop.  Nothing here
imports the oracle or the CUDA package.
"""
from __future__ import annotations

from fractions import Fraction as Fr


class Dual:
    __slots__ = ("v", "t")

    def __init__(self, v, t=0):
        self.v = Fr(v)
        self.t = Fr(t)

    def __add__(self, o):
        o = o if isinstance(o, Dual) else Dual(o)
        return Dual(self.v + o.v, self.t + o.t)

    __radd__ = __add__

    def __mul__(self, o):
        o = o if isinstance(o, Dual) else Dual(o)
        return Dual(self.v * o.v, self.v * o.t + self.t * o.v)

    __rmul__ = __mul__


# ---- primal operators on tuples of scalars (Fraction or Dual) -------------

def op_add(r, a):
    return (r[0] + a[0],)


def op_mul(r, a):
    return (r[0] * a[0],)


def op_min(r, a):  # pick left on ties (reading R3)
    return r if _val(r[0]) <= _val(a[0]) else a


def op_max(r, a):
    return r if _val(r[0]) >= _val(a[0]) else a


def op_linrec(r, a):  # (D, C) (.) (d, c) = (d + c*D, c*C)   (lin_o)
    return (a[0] + a[1] * r[0], a[1] * r[1])


def op_mat2(r, a):  # R . A, row-major 2x2 (scan order of P:1137)
    return (r[0] * a[0] + r[1] * a[2], r[0] * a[1] + r[1] * a[3],
            r[2] * a[0] + r[3] * a[2], r[2] * a[1] + r[3] * a[3])


OPS = {"add": (op_add, 1), "mul": (op_mul, 1), "min": (op_min, 1), "max": (op_max, 1),
       "linrec": (op_linrec, 2), "mat2": (op_mat2, 4)}


def _val(x):
    return x.v if isinstance(x, Dual) else x


def chunk(flat, w):
    return [tuple(flat[i * w:(i + 1) * w]) for i in range(len(flat) // w)]


def scan(op, flat):
    f, w = OPS[op]
    els = chunk(flat, w)
    out = []
    for i, a in enumerate(els):
        out.append(a if i == 0 else f(out[-1], a))
    return [x for e in out for x in e]


def reduce(op, xs):
    f, _ = OPS[op]
    acc = (xs[0],)
    for a in xs[1:]:
        acc = f(acc, (a,))
    return acc[0]


def reduce_by_index(op, m, inds, xs, neutral):
    f, _ = OPS[op]
    hs = [(neutral,) for _ in range(m)]
    for b, a in zip(inds, xs):
        if 0 <= b < m:
            hs[b] = f(hs[b], (a,))
    return [h[0] for h in hs]


def scatter(xs, is_, vs):
    ys = list(xs)
    for j, t in enumerate(is_):
        if 0 <= t < len(xs):
            ys[t] = vs[j]
    return ys


# ---- vjp by forward mode over the standard basis --------------------------

def vjp_by_duals(fn, x, ybar):
    """abar_k = <ybar, J(x) e_k>, J from dual numbers."""
    x = [Fr(v) for v in x]
    out = []
    for k in range(len(x)):
        dx = [Dual(v, 1 if i == k else 0) for i, v in enumerate(x)]
        y = fn(dx)
        y = y if isinstance(y, list) else [y]
        out.append(sum((Fr(yb) * _tan(yi) for yb, yi in zip(ybar, y)), Fr(0)))
    return out


def _tan(y):
    return y.t if isinstance(y, Dual) else Fr(0)


def vjp_by_central_fd(fn, x, ybar, h=Fr(1, 2)):
    """Central difference of <ybar, fn(x)>; exact for multilinear fn (any h)."""
    x = [Fr(v) for v in x]
    out = []
    for k in range(len(x)):
        xp = list(x); xp[k] += h
        xm = list(x); xm[k] -= h
        yp, ym = fn(xp), fn(xm)
        yp = yp if isinstance(yp, list) else [yp]
        ym = ym if isinstance(ym, list) else [ym]
        sp = sum((Fr(b) * v for b, v in zip(ybar, yp)), Fr(0))
        sm = sum((Fr(b) * v for b, v in zip(ybar, ym)), Fr(0))
        out.append((sp - sm) / (2 * h))
    return out
