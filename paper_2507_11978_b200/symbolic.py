"""Integer expressions for grids, offsets and masks.

Same semantics as the reference's ``symexpr`` (symexpr.py:31-322): Python
floor semantics for ``//`` and ``%``, ``ceildiv(a, b) = -((-a) // b)``
(symexpr.py:150-156), a zero divisor is an evaluation error
(symexpr.py:168-173), and a sound local rewriter (constant folding plus the
identity set of symexpr.py:200-246).  The tree layout is the reference's JSON
form (``["add", lhs, rhs]``, ``["sym", name]``, ``["const", k]``,
symexpr.py:251-275) so trees produced by either front end can be compared
structurally and compiled to the C-ABI bytecode (``bytecode.py``).

Expressions are plain immutable tuples underneath (``Expr.node``); ``Expr``
adds operator sugar.  ``from_any`` also accepts the reference's ``SymExpr``
objects by duck typing (``.kind/.value/.name/.args``), which is how a
``CheckedSpec`` built by the reference front end reaches this backend.
"""

from __future__ import annotations

import re
from typing import Mapping, Union

import numpy as np

_IDENT = re.compile(r"[A-Za-z_][A-Za-z0-9_]*\Z")

BINARY = ("add", "sub", "mul", "floordiv", "ceildiv", "mod", "min", "max")
KINDS = ("const", "sym", "neg") + BINARY


class ExprError(Exception):
    """Malformed expression."""


class EvalError(ExprError):
    """Unbound symbol or zero divisor during evaluation."""


class Expr:
    """Immutable integer expression; ``node`` is the JSON-form tuple tree."""

    __slots__ = ("node", "_hash")

    def __init__(self, node):
        object.__setattr__(self, "node", node)
        object.__setattr__(self, "_hash", hash(node))

    def __setattr__(self, k, v):
        raise AttributeError("Expr is immutable")

    # structural identity
    def __eq__(self, other):
        return isinstance(other, Expr) and self.node == other.node

    def __hash__(self):
        return self._hash

    @property
    def kind(self) -> str:
        return self.node[0]

    @property
    def value(self) -> int:
        return self.node[1] if self.node[0] == "const" else 0

    @property
    def name(self) -> str:
        return self.node[1] if self.node[0] == "sym" else ""

    @property
    def args(self) -> tuple["Expr", ...]:
        if self.node[0] in ("const", "sym"):
            return ()
        return tuple(Expr(a) for a in self.node[1:])

    def _bin(self, kind, other, swap=False):
        o = lift(other)
        a, b = (o, self) if swap else (self, o)
        return Expr((kind, a.node, b.node))

    def __add__(self, o):
        return self._bin("add", o)

    def __radd__(self, o):
        return self._bin("add", o, True)

    def __sub__(self, o):
        return self._bin("sub", o)

    def __rsub__(self, o):
        return self._bin("sub", o, True)

    def __mul__(self, o):
        return self._bin("mul", o)

    def __rmul__(self, o):
        return self._bin("mul", o, True)

    def __floordiv__(self, o):
        return self._bin("floordiv", o)

    def __mod__(self, o):
        return self._bin("mod", o)

    def __neg__(self):
        return Expr(("neg", self.node))

    def __repr__(self):
        return f"Expr<{text(self)}>"


def lit(k: int) -> Expr:
    return Expr(("const", int(k)))


def var(name: str) -> Expr:
    if not name or not _IDENT.match(name):
        raise ExprError(f"symbol name must be an identifier, got {name!r}")
    return Expr(("sym", name))


def lift(x) -> Expr:
    if isinstance(x, Expr):
        return x
    if isinstance(x, (int, np.integer)) and not isinstance(x, bool):
        return lit(int(x))
    return from_any(x)


def ceil_div(a, b) -> Expr:
    return Expr(("ceildiv", lift(a).node, lift(b).node))


def emin(a, b) -> Expr:
    return Expr(("min", lift(a).node, lift(b).node))


def emax(a, b) -> Expr:
    return Expr(("max", lift(a).node, lift(b).node))


ZERO = lit(0)
ONE = lit(1)


# --- conversion ----------------------------------------------------------

def _node_from_tree(obj):
    if not isinstance(obj, (list, tuple)) or not obj:
        raise ExprError(f"malformed expression tree: {obj!r}")
    tag = obj[0]
    if tag == "const":
        return ("const", int(obj[1]))
    if tag == "sym":
        if not _IDENT.match(str(obj[1])):
            raise ExprError(f"bad symbol {obj[1]!r}")
        return ("sym", str(obj[1]))
    if tag == "neg":
        if len(obj) != 2:
            raise ExprError("neg takes one operand")
        return ("neg", _node_from_tree(obj[1]))
    if tag in BINARY:
        if len(obj) != 3:
            raise ExprError(f"{tag} takes two operands")
        return (tag, _node_from_tree(obj[1]), _node_from_tree(obj[2]))
    raise ExprError(f"unknown expression tag {tag!r}")


def from_tree(obj) -> Expr:
    """From the JSON list form (reference symexpr.py:259-275)."""
    return Expr(_node_from_tree(obj))


def to_tree(e: Expr):
    def walk(n):
        if n[0] in ("const", "sym"):
            return [n[0], n[1]]
        return [n[0]] + [walk(a) for a in n[1:]]

    return walk(lift(e).node)


def from_any(x) -> Expr:
    """Accept an Expr, an int, a JSON tree, or a reference SymExpr (duck typed)."""
    if isinstance(x, Expr):
        return x
    if isinstance(x, (int, np.integer)) and not isinstance(x, bool):
        return lit(int(x))
    if isinstance(x, (list, tuple)):
        return from_tree(x)
    kind = getattr(x, "kind", None)
    if kind is None:
        raise ExprError(f"cannot interpret {type(x).__name__} as an expression")

    def walk(o):
        k = o.kind
        if k == "const":
            return ("const", int(o.value))
        if k == "sym":
            return ("sym", str(o.name))
        if k == "neg":
            return ("neg", walk(o.args[0]))
        if k in BINARY:
            return (k, walk(o.args[0]), walk(o.args[1]))
        raise ExprError(f"unknown expression kind {k!r}")

    return Expr(walk(x))


# --- queries -------------------------------------------------------------

def symbols(e) -> frozenset:
    out = set()

    def walk(n):
        if n[0] == "sym":
            out.add(n[1])
        elif n[0] != "const":
            for a in n[1:]:
                walk(a)

    walk(lift(e).node)
    return frozenset(out)


def subst(e, mapping: Mapping[str, Union[Expr, int]]) -> Expr:
    m = {k: lift(v).node for k, v in mapping.items()}

    def walk(n):
        if n[0] == "sym":
            return m.get(n[1], n)
        if n[0] == "const":
            return n
        return (n[0],) + tuple(walk(a) for a in n[1:])

    return Expr(walk(lift(e).node))


# --- evaluation ----------------------------------------------------------

def _is_arr(v):
    return isinstance(v, np.ndarray)


def _nonzero_divisor(b):
    if _is_arr(b):
        if np.any(b == 0):
            raise EvalError("division or modulo by zero")
    elif b == 0:
        raise EvalError("division or modulo by zero")


def evaluate(e, env: Mapping[str, object]):
    """Evaluate with ints or int64 numpy arrays bound to the symbols."""

    def walk(n):
        k = n[0]
        if k == "const":
            return n[1]
        if k == "sym":
            try:
                return env[n[1]]
            except KeyError:
                raise EvalError(f"unbound symbol {n[1]!r}") from None
        if k == "neg":
            return -walk(n[1])
        a = walk(n[1])
        b = walk(n[2])
        if k == "add":
            return a + b
        if k == "sub":
            return a - b
        if k == "mul":
            return a * b
        if k == "floordiv":
            _nonzero_divisor(b)
            return a // b
        if k == "ceildiv":
            _nonzero_divisor(b)
            return -((-a) // b)
        if k == "mod":
            _nonzero_divisor(b)
            return a % b
        if k == "min":
            return np.minimum(a, b) if (_is_arr(a) or _is_arr(b)) else min(a, b)
        if k == "max":
            return np.maximum(a, b) if (_is_arr(a) or _is_arr(b)) else max(a, b)
        raise ExprError(f"unknown kind {k!r}")

    return walk(lift(e).node)


# --- simplification --------------------------------------------------------

def _c(n, k=None):
    return n[0] == "const" and (k is None or n[1] == k)


def _step(n):
    """One local rewrite at the root; returns the same object if none applies."""
    k = n[0]
    if k == "neg":
        a = n[1]
        if a[0] == "neg":
            return a[1]
        if a[0] == "const":
            return ("const", -a[1])
        return n
    a, b = n[1], n[2]
    if _c(a) and _c(b) and not (k in ("floordiv", "ceildiv", "mod") and b[1] == 0):
        return ("const", int(evaluate(Expr(n), {})))
    same = a == b and a[0] != "const"
    if k == "add":
        if _c(a, 0):
            return b
        if _c(b, 0):
            return a
    elif k == "sub":
        if _c(b, 0):
            return a
        if same:
            return ZERO.node
    elif k == "mul":
        if _c(a, 1):
            return b
        if _c(b, 1):
            return a
        if _c(a, 0) or _c(b, 0):
            return ZERO.node
    elif k in ("floordiv", "ceildiv"):
        if _c(b, 1):
            return a
        if _c(a, 0) and not _c(b):
            return ZERO.node
        if same:
            return ONE.node
    elif k == "mod":
        if _c(b, 1):
            return ZERO.node
        if _c(a, 0) and not _c(b):
            return ZERO.node
        if same:
            return ZERO.node
    elif k in ("min", "max"):
        if a == b:
            return a
    return n


def _simp(n):
    if n[0] in ("const", "sym"):
        return n
    n = (n[0],) + tuple(_simp(a) for a in n[1:])
    for _ in range(8):
        m = _step(n)
        if m is n:
            return n
        n = m
        if n[0] in ("const", "sym"):
            return n
    return n


def simplify(e) -> Expr:
    """Sound rewrite: same value under every binding; zero divisors kept."""
    return Expr(_simp(lift(e).node))


# --- rendering -------------------------------------------------------------

_PREC = {"add": 10, "sub": 10, "mul": 20, "floordiv": 20, "mod": 20, "neg": 25}
_OPS = {"add": " + ", "sub": " - ", "mul": " * ", "floordiv": " // ", "mod": " % "}


def text(e, cdiv: str = "cdiv", fmin: str = "min", fmax: str = "max") -> str:
    """Infix text; equal-precedence right operands are parenthesised."""

    def r(n, parent):
        k = n[0]
        if k in ("const", "sym"):
            return str(n[1])
        if k in ("ceildiv", "min", "max"):
            fn = {"ceildiv": cdiv, "min": fmin, "max": fmax}[k]
            return f"{fn}({r(n[1], 0)}, {r(n[2], 0)})"
        if k == "neg":
            s = "-" + r(n[1], _PREC["neg"] + 1)
            return f"({s})" if parent > _PREC["neg"] else s
        p = _PREC[k]
        s = r(n[1], p) + _OPS[k] + r(n[2], p + 1)
        return f"({s})" if p < parent else s

    return r(lift(e).node, 0)


# --- canonical form (structural comparison up to algebra) -------------------
#
# Two front ends can build the same map with different association /
# commutation orders (a*(b*c) vs (b*a)*c, x + 0, ...).  ``canonical`` turns an
# expression into a hashable normal form: a polynomial with integer
# coefficients over ATOMS, where an atom is a symbol or a floordiv / ceildiv /
# mod / min / max of two canonical operands.  On top of ring arithmetic it
# applies the exact identities (q*c) // c = q, (q*c) % c = 0 (c a constant
# or a monomial dividing every term; c != 0), x // 1 = x, x % 1 = 0, and
# (x // b) // c = x // (b*c), which assumes positive divisors - true for
# every divisor an arrangement produces (tile sizes and extents).  Equal
# canonical forms imply equal values under every binding with positive
# divisors; the converse is not claimed (the backend only needs "same form
# => same map", and tests check the forms of both front ends agree).

def _padd(p, q, sign=1):
    out = dict(p)
    for m, c in q.items():
        v = out.get(m, 0) + sign * c
        if v:
            out[m] = v
        else:
            out.pop(m, None)
    return out


def _pmul(p, q):
    out: dict = {}
    for m1, c1 in p.items():
        for m2, c2 in q.items():
            m = tuple(sorted(m1 + m2))
            v = out.get(m, 0) + c1 * c2
            if v:
                out[m] = v
            else:
                out.pop(m, None)
    return out


def _pkey(p):
    return tuple(sorted(p.items()))


def _pconst(p):
    if not p:
        return 0
    if len(p) == 1 and () in p:
        return p[()]
    return None


def _atom(kind, pa, pb):
    return {((kind, _pkey(pa), _pkey(pb)),): 1}


def _divide_by_monomial(p, mono):
    """p / mono if mono divides every monomial of p (multiset inclusion)."""
    out = {}
    for m, c in p.items():
        rest = list(m)
        for a in mono:
            if a not in rest:
                return None
            rest.remove(a)
        out[tuple(rest)] = c
    return out


def _poly(n):
    k = n[0]
    if k == "const":
        return {(): n[1]} if n[1] else {}
    if k == "sym":
        return {(("sym", n[1]),): 1}
    if k == "neg":
        return {m: -c for m, c in _poly(n[1]).items()}
    pa, pb = _poly(n[1]), _poly(n[2])
    if k == "add":
        return _padd(pa, pb)
    if k == "sub":
        return _padd(pa, pb, -1)
    if k == "mul":
        return _pmul(pa, pb)
    if k in ("min", "max"):
        ka, kb = _pkey(pa), _pkey(pb)
        if ka == kb:
            return pa
        ca, cb = _pconst(pa), _pconst(pb)
        if ca is not None and cb is not None:
            v = min(ca, cb) if k == "min" else max(ca, cb)
            return {(): v} if v else {}
        lo, hi = sorted((ka, kb))
        return {((k, lo, hi),): 1}
    # floordiv / ceildiv / mod
    ca, cb = _pconst(pa), _pconst(pb)
    if cb is not None and cb != 0:
        if ca is not None:
            v = int(evaluate(Expr((k, ("const", ca), ("const", cb))), {}))
            return {(): v} if v else {}
        if all(c % cb == 0 for c in pa.values()):
            return {} if k == "mod" else {m: c // cb for m, c in pa.items()}
    elif cb is None and len(pb) == 1:
        (mono, coeff), = pb.items()
        if coeff == 1:
            q = _divide_by_monomial(pa, mono)
            if q is not None:
                return {} if k == "mod" else q
    if not pa and (cb is None or cb != 0):
        return {}
    if k == "floordiv" and len(pa) == 1:
        (mono, coeff), = pa.items()
        if coeff == 1 and len(mono) == 1 and mono[0][0] == "floordiv":
            inner = mono[0]
            x, b = dict(inner[1]), dict(inner[2])
            return _poly_floordiv(x, _pmul(b, pb))
    return _atom(k, pa, pb)


def _poly_floordiv(px, pd):
    """Canonical x // d for polynomials (re-enters the floordiv rules)."""
    cd = _pconst(pd)
    if cd is not None and cd != 0 and all(c % cd == 0 for c in px.values()):
        return {m: c // cd for m, c in px.items()}
    return _atom("floordiv", px, pd)


def canonical(e):
    """Hashable normal form of ``e`` (see the block comment above)."""
    return _pkey(_poly(lift(e).node))
