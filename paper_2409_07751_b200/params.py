"""RNS-CKKS parameter sets: prime chain, special primes, canonical scales.

The reference has no modulus chain: its `BackendConfig` collapses rescaling
into an integer `level` (`/root/reference/pkg/src/hekan/backend.py:23-66`,
`SPEC.md` "Rescaling/modulus chains are collapsed into the integer level").
This module supplies the chain that the reference's level maps onto:

* a ciphertext at reference level ``l`` lives modulo ``Q_l = q_0 * ... * q_l``
  (``l + 1`` RNS limbs, limb-major in HBM);
* every multiplication drops ``q_l`` by rescaling, exactly mirroring
  ``level -= 1`` in `HeBackend.slotwise` (`backend.py:215-224`);
* ``q_0`` is ~50 bits and the rescaling primes sit next to the scale
  (~2^46), after the paper's 51/46/51 chain (`PAPER.md:321`); the special
  primes sit just below 2^47 (alpha of them: P / Q_digit >= 2^13). Every prime
  is in (2^44, 2^50) (25-bit split MACs) and all but q_0 are below 2^47, which
  keeps the GPU's float64 NTT free of intra-phase reductions.

Canonical scales. Ciphertexts at level ``l`` always carry scale
``Delta_l``. The chain is built top-down with ``Delta_L = 2^scale_bits`` and
``q_l`` = the NTT-friendly prime closest to ``Delta_l^2 / 2^scale_bits``, so
``Delta_{l-1} = Delta_l^2 / q_l`` stays within ~2^-25 of ``2^scale_bits``
at every level. A ct x ct product of two canonical ciphertexts therefore lands
exactly on the canonical scale of the next level, a plaintext product uses an
encoding scale of ``q_l * Delta_{l-1} / Delta_l``, and level alignment on
add/sub only drops limbs (relative scale mismatch below 1e-7).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

__all__ = ["CkksParams", "is_prime", "make_params", "kan_params",
           "microbench_params"]


def _miller_rabin(n: int) -> bool:
    # deterministic for n < 3.3e24 with these bases
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def is_prime(n: int) -> bool:
    return _miller_rabin(int(n))


def _primitive_2n_root(q: int, two_n: int) -> int:
    """Smallest x^((q-1)/2N) that is a primitive 2N-th root of unity mod q."""
    if (q - 1) % two_n:
        raise ValueError(f"{q} is not 1 mod {two_n}")
    e = (q - 1) // two_n
    for x in range(2, 1 << 20):
        psi = pow(x, e, q)
        if pow(psi, two_n // 2, q) == q - 1:
            # take the minimal primitive root in the cyclic group it generates
            best, cur = psi, psi
            sq = psi * psi % q
            for _ in range(two_n // 2 - 1):
                cur = cur * sq % q  # odd powers are the primitive ones
                if cur < best:
                    best = cur
            return best
    raise ValueError(f"no primitive {two_n}-th root mod {q}")


def _prime_near(target: float, two_n: int, used: set, upper: int | None = None) -> int:
    """NTT-friendly prime (== 1 mod 2N) closest to `target`, not in `used`."""
    base = int(round(target / two_n)) * two_n + 1
    for step in range(0, 1 << 30):
        for cand in ((base + step * two_n, base - step * two_n) if step else (base,)):
            if cand <= two_n or cand in used:
                continue
            if upper is not None and cand >= upper:
                continue
            if is_prime(cand):
                return cand
    raise ValueError("prime search exhausted")


def _primes_below(bound: int, two_n: int, count: int, used: set) -> list:
    out = []
    cand = ((bound - 1) // two_n) * two_n + 1
    while len(out) < count:
        if cand not in used and is_prime(cand):
            out.append(cand)
        cand -= two_n
        if cand <= two_n:
            raise ValueError("prime search exhausted")
    return out


@dataclass(frozen=True)
class CkksParams:
    """Run-time RNS-CKKS parameters (ring degree, chain, keys, scales)."""

    log_n: int
    q: tuple              # ciphertext primes q_0..q_L (L = depth budget)
    p: tuple              # special primes for hybrid key switching
    dnum: int             # key-switching digits over the full chain
    scales: tuple         # canonical scale per level, len L + 1
    psi_q: tuple = field(default=())  # primitive 2N-th roots per q prime
    psi_p: tuple = field(default=())  # ... per special prime
    label: str = ""

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def slot_count(self) -> int:
        return self.n // 2

    @property
    def depth(self) -> int:
        """Reference `depth_budget`: the top level (number of rescales)."""
        return len(self.q) - 1

    @property
    def alpha(self) -> int:
        """Primes per key-switching digit."""
        return -(-len(self.q) // self.dnum)

    @property
    def n_digits(self) -> int:
        return -(-len(self.q) // self.alpha)

    def digits_at(self, level: int) -> int:
        return level // self.alpha + 1

    def scale(self, level: int) -> float:
        return self.scales[level]

    def pt_mult_scale(self, level: int) -> float:
        """Encoding scale of a plaintext multiplied into a level-`level` ct so
        the rescaled product lands on the canonical scale of level - 1."""
        return self.q[level] * self.scales[level - 1] / self.scales[level]

    @property
    def log_pq(self) -> float:
        """log2 of the whole modulus Q * P (the number security is read from)."""
        return sum(math.log2(x) for x in list(self.q) + list(self.p))

    def describe(self) -> str:
        qb = [round(math.log2(x), 2) for x in self.q]
        pb = [round(math.log2(x), 2) for x in self.p]
        return (f"N=2^{self.log_n} L={self.depth} dnum={self.dnum} alpha={self.alpha} "
                f"q bits={qb[0]}/{qb[1] if len(qb) > 1 else '-'}.. p bits={pb[:2]}.. "
                f"logQP={sum(math.log2(x) for x in self.q + self.p):.1f}")

    def to_json(self) -> dict:
        return {"log_n": self.log_n, "q": list(self.q), "p": list(self.p),
                "dnum": self.dnum, "scales": list(self.scales), "label": self.label}


def make_params(log_n: int, depth: int, scale_bits: int = 46, q0_bits: int = 50,
                special_bits: int = 47, dnum: int = 3, n_special: int | None = None,
                label: str = "") -> CkksParams:
    """Scale-stable chain: q_0 just below 2^q0_bits, rescaling primes chosen
    top-down so the canonical scale never drifts from 2^scale_bits."""
    if not 3 <= log_n <= 17:
        raise ValueError("log_n must be in [3, 17]")
    if depth < 0:
        raise ValueError("depth must be >= 0")
    two_n = 2 << log_n
    used: set = set()
    target = float(2 ** scale_bits)
    scales = [0.0] * (depth + 1)
    q = [0] * (depth + 1)
    scales[depth] = target
    for lvl in range(depth, 0, -1):
        want = scales[lvl] * scales[lvl] / target
        q[lvl] = _prime_near(want, two_n, used, upper=1 << q0_bits)
        used.add(q[lvl])
        scales[lvl - 1] = scales[lvl] * scales[lvl] / q[lvl]
    q[0] = _primes_below(1 << q0_bits, two_n, 1, used)[0]
    used.add(q[0])
    dnum = max(1, min(dnum, depth + 1))
    alpha = -(-(depth + 1) // dnum)
    if n_special is None:
        n_special = alpha
    p = _primes_below(1 << special_bits, two_n, n_special, used)
    return CkksParams(log_n=log_n, q=tuple(q), p=tuple(p), dnum=dnum,
                      scales=tuple(scales),
                      psi_q=tuple(_primitive_2n_root(x, two_n) for x in q),
                      psi_p=tuple(_primitive_2n_root(x, two_n) for x in p),
                      label=label)


def kan_params(depth: int, log_n: int = 16, dnum: int = 3) -> CkksParams:
    """Encrypted-KAN chain (paper-style 50/46/50 bits, `PAPER.md:321`)."""
    return make_params(log_n, depth, scale_bits=46, q0_bits=50, special_bits=47,
                       dnum=dnum, label=f"kan-L{depth}")


def microbench_params(log_n: int = 16, limbs: int = 24, dnum: int = 3) -> CkksParams:
    """BASELINE config 2: 24 ~50-bit limbs, hybrid dnum=3 (alpha = 8 special
    primes; SURVEY §0.6 explains why one special prime cannot cover a digit)."""
    two_n = 2 << log_n
    used: set = set()
    q = _primes_below(1 << 50, two_n, limbs, used)
    used.update(q)
    alpha = -(-limbs // dnum)
    p = _primes_below(1 << 50, two_n, alpha, used)
    scales = tuple(float(2 ** 40) for _ in q)
    return CkksParams(log_n=log_n, q=tuple(q), p=tuple(p), dnum=dnum, scales=scales,
                      psi_q=tuple(_primitive_2n_root(x, two_n) for x in q),
                      psi_p=tuple(_primitive_2n_root(x, two_n) for x in p),
                      label=f"micro-{limbs}x50")
