"""TEST INFRASTRUCTURE ONLY — exact first-contact times of CCD queries.

Restates the reference's exact-rational oracle (proj/src/oracle.cpp, which needs
Boost.Multiprecision + GMP and does not build here) with Python Fractions and
sympy's exact real-root isolation, to check the narrow phase's conservativeness
("zero false negatives") against ground truth rather than only against the
reference implementation:

* trajectory / build_polys (oracle.cpp:285-331): every coordinate is linear in t,
  x(t) = x0 + t (x1 - x0) with exact rationals; VF: coplanarity cubic
  w . (e1 x e2), Gram denominator a c - b^2 and barycentric numerators
  u = d c - e b, v = a e - b d; EE: r . (d1 x d2), |d1 x d2|^2 and
  u = (r x d2) . n, v = (r x d1) . n;
* classify_uv / validity_at (oracle.cpp:335-361): exact interval evaluation of
  the denominator and numerators over a root's isolating interval, Valid /
  Invalid / Unknown;
* roots in [0, 1] in increasing order (oracle.cpp:371-453 isolates with Sturm
  chains; sympy's Poly.intervals does the same job exactly), each refined until
  validity is decided (oracle_toi, oracle.cpp:626-691).

exact_first_contact(kind, points) returns (status, lo, hi): status "contact"
with the first valid root bracketed in [lo, hi], "none" (no valid root in
[0, 1]), or "indeterminate" (identically coplanar motion, or a root whose
validity stays undecided — degenerate configurations the reference oracle also
treats separately).
"""
from __future__ import annotations

from fractions import Fraction

import sympy

_t = sympy.Symbol("t")


def _traj(points, p):
    """[(x0_c, dx_c)] exact, point p of a 24-double record (reference order)."""
    out = []
    for c in range(3):
        x0 = Fraction(float(points[3 * p + c]))
        x1 = Fraction(float(points[12 + 3 * p + c]))
        out.append((x0, x1 - x0))
    return out


def _poly(v):
    """linear (a, b) -> sympy Poly a + b t over QQ."""
    a, b = v
    return sympy.Poly(sympy.Rational(b.numerator, b.denominator) * _t
                      + sympy.Rational(a.numerator, a.denominator), _t, domain="QQ")


def _vec(tr):
    return [_poly(x) for x in tr]


def _sub(a, b):
    return [x - y for x, y in zip(a, b)]


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def build_polys(kind: int, points):
    """oracle.cpp:300-331 (kind 0 = vertex-face, 1 = edge-edge)."""
    p = [_vec(_traj(points, i)) for i in range(4)]
    if kind == 0:
        e1, e2, w = _sub(p[2], p[1]), _sub(p[3], p[1]), _sub(p[0], p[1])
        cop = _dot(w, _cross(e1, e2))
        a, b, c = _dot(e1, e1), _dot(e1, e2), _dot(e2, e2)
        d, e = _dot(w, e1), _dot(w, e2)
        return cop, a * c - b * b, d * c - e * b, a * e - b * d
    d1, d2, r = _sub(p[1], p[0]), _sub(p[3], p[2]), _sub(p[2], p[0])
    n = _cross(d1, d2)
    return _dot(r, n), _dot(n, n), _dot(_cross(r, d2), n), _dot(_cross(r, d1), n)


def _eval_interval(poly, lo: Fraction, hi: Fraction):
    """Exact bounds of poly over [lo, hi] (interval Horner on rationals)."""
    coeffs = [Fraction(int(c.p), int(c.q)) for c in poly.all_coeffs()]
    rlo = rhi = Fraction(0)
    for c in coeffs:
        prods = [rlo * lo, rlo * hi, rhi * lo, rhi * hi]
        rlo, rhi = min(prods) + c, max(prods) + c
    return rlo, rhi


def _divide(n, d):
    q = [n[0] / d[0], n[0] / d[1], n[1] / d[0], n[1] / d[1]]
    return min(q), max(q)


def _validity(kind, polys, lo, hi):
    """oracle.cpp:335-361."""
    _, den, un, vn = polys
    d = _eval_interval(den, lo, hi)
    if d[0] <= 0 <= d[1]:
        return "unknown"
    u = _divide(_eval_interval(un, lo, hi), d)
    v = _divide(_eval_interval(vn, lo, hi), d)
    if kind == 0:
        if u[0] >= 0 and v[0] >= 0 and u[1] + v[1] <= 1:
            return "valid"
        if u[1] < 0 or v[1] < 0 or u[0] + v[0] > 1:
            return "invalid"
        return "unknown"
    if u[0] >= 0 and u[1] <= 1 and v[0] >= 0 and v[1] <= 1:
        return "valid"
    if u[1] < 0 or u[0] > 1 or v[1] < 0 or v[0] > 1:
        return "invalid"
    return "unknown"


def _fr(x):
    return Fraction(int(x.p), int(x.q))


def _sr(f: Fraction):
    return sympy.Rational(f.numerator, f.denominator)


def exact_first_contact(kind: int, points, max_refine: int = 60, width=Fraction(1, 1 << 80)):
    polys = build_polys(int(kind), points)
    cop = polys[0]
    if cop.is_zero:
        return "indeterminate", None, None
    # square-free part: same roots, each simple, so isolating intervals can be
    # refined by bisection (the reference's Sturm-chain isolation, oracle.cpp:371-453)
    sf = cop.sqf_part()
    for (slo, shi), _mult in sorted(sf.intervals(inf=0, sup=1), key=lambda r: r[0][0]):
        lo, hi = _fr(slo), _fr(shi)
        v = "unknown"
        for _ in range(max_refine):
            v = _validity(kind, polys, lo, hi)
            if v != "unknown" or lo == hi:
                break
            a, b = sf.refine_root(_sr(lo), _sr(hi), eps=_sr((hi - lo) / 4))
            lo, hi = _fr(a), _fr(b)
        if v == "valid":
            if hi - lo > width:
                a, b = sf.refine_root(_sr(lo), _sr(hi), eps=_sr(width))
                lo, hi = _fr(a), _fr(b)
            return "contact", lo, hi
        if v == "unknown":
            return "indeterminate", lo, hi
    return "none", None, None
