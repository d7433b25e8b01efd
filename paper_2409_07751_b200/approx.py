"""HE polynomial evaluation and the composite-sign comparator: engine deltas.

The reference side of `/root/reference/pkg/src/hekan/approx.py` is imported,
not restated: `Polynomial`, `ApproxRange`, `WeightScheme`, the range
estimators and fitters (`estimate_range`, `fit_weighted_ls`, `fit_ols`,
`fit_remez`), `poly_eval_depth`, `eval_poly_clear`, `poly_comp_clear` and the
comparator fitter `build_composite_sign` (its stages are fitted by the
reference's own Remez code). What lives here is what the RNS-CKKS engine runs
differently:

* `_estrin` keeps the reference's balanced power tree (approx.py:369-405) —
  same tree, same counts, same levels — and folds each four-coefficient block
  whose low half is a leaf (`c1 x + c0`) into the relinearised product that
  consumes it (`HeBackend.mul_lin`: one rescale instead of two);
* the comparator stages are the reference's polynomials re-expanded exactly
  over Chebyshev T_k (|c| <= 1.3 instead of monomials up to 6e10, SURVEY
  §0.4, which diverge under real CKKS noise) and evaluated with the same tree
  shape, so levels and multiplication counts are unchanged; each squaring is
  T_2k = 2 T_k^2 - 1 (`HeBackend.mul_affine`, one product);
* SiLU fits whose monomial intermediates blow up (c3's degree 63) run as the
  same polynomial in T_k on the fit interval (+1 level off the critical path).
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from ._ref import hekan
from .errors import InputOutOfRange

_ha = hekan.approx
Polynomial = _ha.Polynomial
ApproxRange = _ha.ApproxRange
WeightScheme = _ha.WeightScheme
range_from_moments = _ha.range_from_moments
estimate_range = _ha.estimate_range
fit_weighted_ls = _ha.fit_weighted_ls
fit_ols = _ha.fit_ols
fit_remez = _ha.fit_remez
poly_eval_depth = _ha.poly_eval_depth
eval_poly_clear = _ha.eval_poly_clear
poly_comp_clear = _ha.poly_comp_clear
_ArrayOps = _ha._ArrayOps
_trimmed = _ha._trimmed


# ---------------------------------------------------------------------------
# balanced power tree on the engine (approx.py:311-418)
# ---------------------------------------------------------------------------


class _HeOps(_ha._HeOps):
    """The reference adapter (approx.py:311-332) plus the engine's fused
    combines; public constants are trivial encryptions batched like x."""

    def mul_lin(self, a, b, x, k):
        return self.be.mul_lin(a, b, x, k)

    def mul_affine(self, a, b, mult, c):
        return self.be.mul_affine(a, b, mult, c)

    def const(self, c):
        rows = np.full((getattr(self.x, "batch", 1), self.be.config.slot_count), c)
        return self.be.encrypt(rows if getattr(self.x, "batched", False) else rows[0], self.x.level)


def _fusable(ops, method: str) -> bool:
    return hasattr(ops, method) and hasattr(getattr(ops.x, "backend", None), method)


def _combine(ops, xpow, lo_val, hi_val):
    """hi * xpow + lo with the reference's float/zero short-cuts (approx.py:393-403)."""
    if isinstance(hi_val, float):
        term = None if hi_val == 0.0 else ops.mul_const(xpow, hi_val)
    else:
        term = ops.mul(xpow, hi_val)
    if term is None:
        return lo_val
    if isinstance(lo_val, float):
        return term if lo_val == 0.0 else ops.add_const(term, lo_val)
    return ops.add(term, lo_val)


def _fused_combine(ops, xpow, x, c0: float, c1: float, hi_val):
    """hi * xpow + (c1 x + c0) as one relinearised product (`mul_lin`) plus the
    constant: the counts of _combine's mul_const, mul, add, add_const."""
    t = ops.mul_lin(xpow, hi_val, x, c1)
    return t if c0 == 0.0 else ops.add_const(t, float(c0))


def _power_tree(ops, padded: np.ndarray, pows: list, split):
    """Shared recursion of the monomial and Chebyshev trees. `split(c)` maps a
    block's 2h coefficients to (low, high) with p = high * P_h + low."""
    fuse = _fusable(ops, "mul_lin")

    def block(c: np.ndarray):
        if len(c) == 1:
            return float(c[0])
        lo_c, hi_c = split(c)
        if fuse and len(c) == 4 and lo_c[1] != 0.0:
            hi_val = block(hi_c)
            if not isinstance(hi_val, float):
                return _fused_combine(ops, pows[1], pows[0], float(lo_c[0]), float(lo_c[1]), hi_val)
            return _combine(ops, pows[1], block(lo_c), hi_val)
        lo_val = block(lo_c)
        hi_val = block(hi_c)
        return _combine(ops, pows[(len(c) // 2).bit_length() - 1], lo_val, hi_val)

    out = block(padded)
    # `block` is a recursive closure (a reference cycle through its own cell):
    # drop it and the powers so the ciphertexts free now, not at the next gc pass
    del block
    pows.clear()
    return ops.const(out) if isinstance(out, float) else out


def _padded(coeffs: np.ndarray):
    n = len(coeffs)
    m = max(1, (n - 1).bit_length())
    padded = np.zeros(1 << m)
    padded[:n] = coeffs
    return padded, m


def _mono_split(c: np.ndarray):
    h = len(c) // 2
    return c[:h], c[h:]


def _estrin(ops, coeffs: np.ndarray):
    """The reference's balanced power tree over monomials (ceil(log2 n) levels)."""
    n = len(coeffs)
    if n == 1 or (n > 0 and not np.any(coeffs[1:])):
        return ops.const(float(coeffs[0]))
    padded, m = _padded(coeffs)
    pows = [ops.x]
    for _ in range(m - 1):
        pows.append(ops.mul(pows[-1], pows[-1]))
    return _power_tree(ops, padded, pows, _mono_split)


def eval_poly_he(a, p):
    """Reference program (monomial Estrin, approx.py:416-418) on the engine."""
    return _estrin(_HeOps(a), _trimmed(p.coeffs))


# ---------------------------------------------------------------------------
# Chebyshev-basis power tree (same shape, T_{2^k} instead of x^{2^k})
# ---------------------------------------------------------------------------


def _cheb_split(c: np.ndarray):
    """p = q T_h + r for p = sum c_i T_i over 2h coefficients, by
    T_{h+j} = 2 T_h T_j - T_{h-j}; returns (r, q)."""
    h = len(c) // 2
    q = np.zeros(h)
    r = np.array(c[:h], dtype=float)
    q[0] = c[h]
    for j in range(1, h):
        q[j] = 2.0 * c[h + j]
        r[h - j] -= c[h + j]
    return r, q


def _cheb_tree(ops, coeffs: np.ndarray):
    """sum c_k T_k(x) with the Estrin tree shape: ceil(log2 n) levels and the
    ct/pt multiplication counts `_estrin` has on the same sparsity."""
    n = len(coeffs)
    if n == 1 or (n > 0 and not np.any(coeffs[1:])):
        return ops.const(float(coeffs[0]))
    padded, m = _padded(coeffs)
    tpows = [ops.x]
    affine = _fusable(ops, "mul_affine")
    for _ in range(m - 1):
        if affine:  # T_2k = 2 T_k^2 - 1 in the product's epilogue (bit-identical)
            tpows.append(ops.mul_affine(tpows[-1], tpows[-1], 2, -1.0))
            continue
        sq = ops.mul(tpows[-1], tpows[-1])
        tpows.append(ops.add_const(ops.add(sq, sq), -1.0))
    return _power_tree(ops, padded, tpows, _cheb_split)


def _cheb_from_exact(qc) -> np.ndarray:
    """Exact monomial coefficients (Fractions) -> Chebyshev coefficients."""
    n = len(qc)
    T = [[Fraction(1)], [Fraction(0), Fraction(1)]]
    for k in range(2, n):
        a = [Fraction(0)] + [2 * v for v in T[k - 1]]
        b = T[k - 2] + [Fraction(0)] * (len(a) - len(T[k - 2]))
        T.append([x - y for x, y in zip(a, b)])
    rem = list(qc)
    out = [Fraction(0)] * n
    for k in range(n - 1, -1, -1):
        if rem[k] == 0:
            continue
        ck = rem[k] / T[k][k]
        out[k] = ck
        for i in range(k + 1):
            rem[i] -= ck * T[k][i]
    return np.array([float(v) for v in out])


def mono_to_cheb(mono, h: float = 1.0, out_scale: float = 1.0) -> np.ndarray:
    """c with sum c_k T_k(y) == p(h y) / out_scale exactly, for the (exactly
    represented) monomial coefficients of p."""
    hF, sF = Fraction(h), Fraction(out_scale)
    return _cheb_from_exact([Fraction(float(a)) * hF ** i / sF for i, a in enumerate(mono)])


def mono_to_cheb_affine(mono, lo: float, hi: float) -> np.ndarray:
    """c with sum c_k T_k(u) == p(x) for x = (u (hi - lo) + lo + hi) / 2, exactly."""
    coef = [Fraction(float(v)) for v in mono]
    n = len(coef)
    half, mid = (Fraction(hi) - Fraction(lo)) / 2, (Fraction(hi) + Fraction(lo)) / 2
    qc = [coef[-1]] + [Fraction(0)] * (n - 1)  # Horner over polynomials in u
    for i in range(n - 2, -1, -1):
        nq = [Fraction(0)] * n
        for k in range(n - 1):
            nq[k + 1] += qc[k] * half
            nq[k] += qc[k] * mid
        nq[0] += coef[i]
        qc = nq
    return _cheb_from_exact(qc)


@dataclass(frozen=True)
class ChebPoly:
    """p(x) evaluated as sum c_k T_k(x / h) / out_scale, x in [-h, h]."""

    coeffs: tuple
    h: float = 1.0
    out_scale: float = 1.0

    @property
    def degree(self) -> int:
        return len(_trimmed(self.coeffs)) - 1


def eval_cheb_he(a, p: ChebPoly):
    """Encrypted Chebyshev evaluation; the caller supplies x / h in [-1, 1]."""
    return _cheb_tree(_HeOps(a), _trimmed(p.coeffs))


def eval_cheb_clear(p: ChebPoly, y: np.ndarray) -> np.ndarray:
    return _cheb_tree(_ArrayOps(np.asarray(y, dtype=float)), _trimmed(p.coeffs))


# ---------------------------------------------------------------------------
# SiLU activation: reference program or Chebyshev on its fit interval
# ---------------------------------------------------------------------------
# The reference's Estrin program carries intermediates up to sum_k |c_k| M^k
# (M = max |x| over the fit interval); CKKS error is relative to those
# magnitudes, so above this bound the program is unusable under encryption
# (c3's degree-63 fits reach |c| = 9e31 and M^63 = 2^63). Such
# polynomials run as sum c_k T_k(u), u = (2x - lo - hi) / (hi - lo), with the
# exact rational re-expansion of the same polynomial over its fit interval.
CHEB_MAGNITUDE_LIMIT = 1e3


def silu_interval(layer) -> tuple:
    """The SiLU fit interval: the layer's `fit_range` when it records one,
    else the reference's act_stats window mu +/- 5 sigma (approx.py:111-126)."""
    fr = getattr(layer, "fit_range", None)
    if fr is not None:
        return tuple(float(v) for v in fr)
    mu, sigma = layer.act_stats
    return (mu - 5.0 * sigma, mu + 5.0 * sigma)


def silu_uses_cheb(layer) -> bool:
    lo, hi = silu_interval(layer)
    M = max(abs(lo), abs(hi))
    mag = sum(abs(c) * M ** k for k, c in enumerate(layer.silu_poly.coeffs))
    return mag > CHEB_MAGNITUDE_LIMIT


@functools.lru_cache(maxsize=256)
def _silu_cheb_cached(coeffs: tuple, lo: float, hi: float) -> tuple:
    return tuple(mono_to_cheb_affine(coeffs, lo, hi))


def silu_affine(layer) -> tuple:
    lo, hi = silu_interval(layer)
    return 2.0 / (hi - lo), -(lo + hi) / (hi - lo)


def _silu_cheb_coeffs(layer) -> np.ndarray:
    lo, hi = silu_interval(layer)
    return _trimmed(np.array(_silu_cheb_cached(tuple(layer.silu_poly.coeffs), lo, hi)))


def eval_silu_he(ct, layer):
    """SiLU polynomial of `layer` under encryption: the reference program for
    well-conditioned fits, else Chebyshev on the fit interval (+1 level)."""
    if not silu_uses_cheb(layer):
        return eval_poly_he(ct, layer.silu_poly)
    be = ct.backend
    a, b = silu_affine(layer)
    u = be.add(be.mul(ct, a), b)
    return _cheb_tree(_HeOps(u), _silu_cheb_coeffs(layer))


def eval_silu_cheb_clear(layer, x: np.ndarray) -> np.ndarray:
    a, b = silu_affine(layer)
    u = np.asarray(x, dtype=float) * a + b
    return _cheb_tree(_ArrayOps(u), _silu_cheb_coeffs(layer))


def silu_depth(layer) -> int:
    return poly_eval_depth(layer.silu_poly) + (1 if silu_uses_cheb(layer) else 0)


# ---------------------------------------------------------------------------
# composite-polynomial comparison (approx.py:431-534)
# ---------------------------------------------------------------------------


def _bound_up(v: float) -> float:
    """A tidy upper bound (multiple of 1/64) for a stage's output range."""
    return math.ceil(v * 64.0 + 1.0) / 64.0


@dataclass(frozen=True)
class CompositeSign(_ha.CompositeSign):
    """The reference's composite sign (approx.py:431-458: same stages, depth,
    delta, clear schedule) carrying its Chebyshev re-expansion `cheb`: stage k
    reads y_k = x_k / h_k in [-1, 1] and emits p_k(x_k) / h_{k+1}
    (h_0 = h_K = 1)."""

    cheb: tuple = field(default=(), compare=False)

    def __post_init__(self):
        if not self.cheb:
            object.__setattr__(self, "cheb", _cheb_stages(self.stages))

    def apply_cheb_clear(self, y: np.ndarray) -> np.ndarray:
        """Plaintext twin of the encrypted (Chebyshev) schedule."""
        s = np.asarray(y, dtype=float)
        for cp in self.cheb:
            s = eval_cheb_clear(cp, s)
        return s

    def cheb_schedule(self) -> "ChebSchedule":
        return ChebSchedule(self)


class ChebSchedule:
    """A comparator view whose `apply_clear` is the Chebyshev schedule, so the
    reference's cleartext twins (`poly_comp_clear`, `basis_clear`,
    `layer_forward_plain(mode="mirrored")`) mirror what the engine runs."""

    def __init__(self, cs: CompositeSign):
        self.cs = cs
        self.stages = cs.stages
        self.delta = cs.delta

    def depth(self) -> int:
        return self.cs.depth()

    def apply_clear(self, y):
        return self.cs.apply_cheb_clear(y)


def _cheb_stages(stages) -> tuple:
    out = []
    h = 1.0
    grid = np.linspace(-1.0, 1.0, 1 << 16)
    for idx, st in enumerate(stages):
        last = idx == len(stages) - 1
        h_next = 1.0 if last else _bound_up(float(np.max(np.abs(st(h * grid)))))
        out.append(ChebPoly(tuple(mono_to_cheb(st.coeffs, h=h, out_scale=h_next)), h, h_next))
        h = h_next
    return tuple(out)


@functools.lru_cache(maxsize=None)
def build_composite_sign(alpha: float = 7.0, target_eps: float = 2.0 ** -10) -> CompositeSign:
    """The reference fitter's comparator (approx.py:479-508) with its
    Chebyshev re-expansion attached."""
    ref = _ha.build_composite_sign(alpha, target_eps)
    return CompositeSign(ref.stages, ref.precision_alpha, ref.target_eps)


def as_engine_comparator(cs):
    """A reference `CompositeSign` (or ours) as the engine's Chebyshev one."""
    if isinstance(cs, CompositeSign) or not isinstance(cs, _ha.CompositeSign):
        return cs
    return CompositeSign(cs.stages, cs.precision_alpha, cs.target_eps)


def poly_comp(a, b, cs, check_range: bool = False):
    """step(a - b) under encryption: ~1 for a > b, ~0 for a < b, 1/2 at ties
    (approx.py:511-528), the stages run in the Chebyshev basis."""
    cs = as_engine_comparator(cs)
    be = a.backend
    d = be.sub(a, b)
    if check_range:
        vals = np.asarray(d.slots)
        if np.max(np.abs(vals)) > 1.0 + 1e-12:
            raise InputOutOfRange(f"comparator operand out of [-1, 1]: max |d| = {np.max(np.abs(vals))}")
    s = d
    for cp in cs.cheb:
        s = eval_cheb_he(s, cp)
    s = be.add(s, 1.0)
    return be.mul(s, 0.5)


def poly_comp_cheb_clear(d: np.ndarray, cs: CompositeSign) -> np.ndarray:
    """Twin of the encrypted (Chebyshev) comparator schedule."""
    return poly_comp_clear(d, ChebSchedule(as_engine_comparator(cs)))
