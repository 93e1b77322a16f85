"""Filter configuration types, mirroring the reference interface.

Same names, fields, defaults, text grammar and ``ValueError`` cases as the
reference's ``dirfilt.filters`` spec types (reference
``pkg/src/dirfilt/filters.py:34-217``) and constants of
``dirfilt.distance`` (``distance.py:24-30,69-78``), so callers of the
reference's ``apply_filter`` can switch packages without touching their
spec-building code.  Reference objects are also accepted wherever these are
(duck typing on the attribute names).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

FAMILIES = ("identity", "vmf", "bvdf", "ddf", "acwddf")

# Affine chromaticity -> radians calibration (paper Eq. 10; distance.py:29-30).
CALIBRATION_SLOPE = 1.436437
CALIBRATION_INTERCEPT = 0.027664

# Paper Table 1: minimax polynomials a_0..a_q.
# "asin" rows approximate 2*asin(tau/sqrt(2)) for tau = sqrt(1-z) on
# [0, 1/sqrt(2)]; "acos" rows approximate acos(z) on [0, 1/2].
ASIN_COEFFICIENTS = {
    2: (1.830987519e-03, (1.829125e-03, 1.371117, 1.480266e-01)),
    3: (1.358426903e-04, (-1.358425e-04, 1.419488, -3.090315e-02, 1.666491e-01)),
    4: (2.097813673e-05, (2.097797e-05, 1.412840, 1.429881e-02, 6.704361e-02, 6.909677e-02)),
}
ACOS_COEFFICIENTS = {
    2: (9.154936808e-04, (1.569882, -9.695260e-01, -1.480266e-01)),
    3: (6.792158693e-05, (1.570864, -1.003730, 3.090318e-02, -2.356775e-01)),
    4: (1.048948667e-05, (1.570786, -9.990285e-01, -1.429899e-02, -9.481335e-02, -1.381942e-01)),
}

_KINDS = ("exact", "minimax", "chromaticity")
_TOKEN_OF_KIND = {"exact": "exact", "minimax": "minimax", "chromaticity": "rgb"}


@dataclass(frozen=True)
class MinimaxPoly:
    """Polynomial a_0 + a_1 z + ... + a_q z^q with its stated error bound."""

    degree: int
    coefficients: tuple
    domain: tuple
    bound: float

    def __post_init__(self) -> None:
        if len(self.coefficients) != self.degree + 1:
            raise ValueError(f"degree {self.degree} requires {self.degree + 1} coefficients, "
                             f"{len(self.coefficients)} given")
        lo, hi = self.domain
        if not lo < hi:
            raise ValueError(f"empty domain {self.domain}")
        if not self.bound > 0:
            raise ValueError("error bound must be positive")

    def __call__(self, z: float) -> float:
        acc = self.coefficients[self.degree]
        for k in range(self.degree - 1, -1, -1):
            acc = acc * z + self.coefficients[k]
        return acc


@dataclass(frozen=True)
class FastAcosTable:
    """The ACOS/ASIN polynomial pair of one degree q."""

    acos_poly: MinimaxPoly
    asin_poly: MinimaxPoly

    def __post_init__(self) -> None:
        if abs(self.asin_poly.coefficients[1] - math.sqrt(2.0)) > 0.05:
            raise ValueError("asin polynomial slope a_1 must be close to sqrt(2)")
        if abs(self.acos_poly.coefficients[0] - math.pi / 2) > 0.01:
            raise ValueError("acos polynomial constant a_0 must be close to pi/2")

    @property
    def degree(self) -> int:
        return self.acos_poly.degree

    @property
    def max_error(self) -> float:
        return max(self.acos_poly.bound, self.asin_poly.bound)

    @classmethod
    def for_degree(cls, q: int = 4) -> "FastAcosTable":
        if q not in ASIN_COEFFICIENTS:
            raise ValueError(f"minimax degree {q} unavailable (2, 3 or 4)")
        bs, cs = ASIN_COEFFICIENTS[q]
        ba, ca = ACOS_COEFFICIENTS[q]
        return cls(acos_poly=MinimaxPoly(q, ca, (0.0, 0.5), ba),
                   asin_poly=MinimaxPoly(q, cs, (0.0, 1.0 / math.sqrt(2.0)), bs))


@dataclass(frozen=True)
class DirectionalStrategy:
    """How the angular ordering term is evaluated: ``exact`` (arccos),
    ``minimax`` (Table 1 polynomials of degree q) or ``chromaticity``
    (L_p distance of x/sum(x); calibration only in the ACWDDF switch)."""

    kind: str = "exact"
    q: int = 4
    slope: float = CALIBRATION_SLOPE
    intercept: float = CALIBRATION_INTERCEPT

    def __post_init__(self) -> None:
        if self.kind not in _KINDS:
            raise ValueError(f"unknown strategy kind {self.kind!r}")
        if self.kind == "minimax" and self.q not in (2, 3, 4):
            raise ValueError(f"minimax degree must be 2, 3, or 4, got {self.q}")
        if self.kind == "chromaticity" and not self.slope > 0:
            raise ValueError("calibration slope must be positive")

    @classmethod
    def exact(cls) -> "DirectionalStrategy":
        return cls("exact")

    @classmethod
    def minimax(cls, q: int = 4) -> "DirectionalStrategy":
        return cls("minimax", q=q)

    @classmethod
    def chromaticity_calibrated(cls, slope: float = CALIBRATION_SLOPE,
                                intercept: float = CALIBRATION_INTERCEPT) -> "DirectionalStrategy":
        return cls("chromaticity", slope=slope, intercept=intercept)

    @property
    def table(self) -> Optional[FastAcosTable]:
        return FastAcosTable.for_degree(self.q) if self.kind == "minimax" else None

    @property
    def token(self) -> str:
        return _TOKEN_OF_KIND[self.kind]


def center_weight(n: int, k: int) -> int:
    """Centre-pixel weight n - 2k + 2 at smoothing level k in [1, (n+1)/2]."""
    d = (n + 1) // 2
    if k < 1 or k > d:
        raise ValueError(f"smoothing level k must be in [1, {d}], got {k}")
    return n - 2 * k + 2


@dataclass(frozen=True)
class AcwddfParams:
    """ACWDDF switching parameters (lambda, T) and its Minkowski order."""

    lam: int = 2
    threshold: float = 10.8
    p: float = 2.0

    def __post_init__(self) -> None:
        if self.lam < 1:
            raise ValueError(f"lambda must be >= 1, got {self.lam}")
        if self.threshold < 0:
            raise ValueError(f"threshold must be nonnegative, got {self.threshold}")
        if not self.p >= 1.0:
            raise ValueError(f"Minkowski order must be >= 1, got {self.p}")

    def validate_for(self, n: int) -> None:
        d = (n + 1) // 2
        if self.lam + 2 > d:
            raise ValueError(f"lambda {self.lam} needs smoothing levels up to {self.lam + 2}; "
                             f"a window of {n} vectors has d = {d}")


@dataclass(frozen=True)
class FilterSpec:
    """One filter: family, angular strategy, Minkowski order p, window side,
    and ACWDDF parameters (present exactly for the acwddf family)."""

    family: str
    strategy: DirectionalStrategy = field(default_factory=DirectionalStrategy.exact)
    p: float = 2.0
    window: int = 3
    acwddf: Optional[AcwddfParams] = None

    def __post_init__(self) -> None:
        if self.family not in FAMILIES:
            raise ValueError(f"unknown filter family {self.family!r} (choose from {FAMILIES})")
        if not self.p >= 1.0:
            raise ValueError(f"Minkowski order must be >= 1, got {self.p}")
        if self.window < 3 or self.window % 2 == 0:
            raise ValueError(f"window side must be odd and >= 3, got {self.window}")
        if (self.acwddf is not None) != (self.family == "acwddf"):
            raise ValueError("acwddf parameters are required exactly when family is acwddf")
        if self.acwddf is not None:
            self.acwddf.validate_for(self.window * self.window)

    @property
    def name(self) -> str:
        if self.family == "identity":
            return "identity"
        out = [self.family]
        if self.family != "vmf":
            out.append(self.strategy.token)
            if self.strategy.kind == "minimax":
                out.append(f"q={self.strategy.q}")
        if self.p != 2.0:
            out.append(f"p={_num(self.p)}")
        if self.window != 3:
            out.append(f"window={self.window}")
        if self.acwddf is not None:
            out.append(f"lambda={self.acwddf.lam}")
            out.append(f"T={_num(self.acwddf.threshold)}")
        return ":".join(out)

    def __str__(self) -> str:
        return self.name


CW_FAMILIES = ("cwvmf", "cwddf")


@dataclass(frozen=True)
class CenterWeightedSpec:
    """Extension: the reference's window-level
    centre-weighted filters applied to every window of an image --
    ``cwvmf(w, k, p)`` (reference filters.py:331-337, weighted Minkowski sums
    only) and ``cwddf(w, k, p, strategy)`` (filters.py:304-328, weighted
    angular x Minkowski sums).  ``k`` is the smoothing level of
    ``center_weight(n, k)``: k = 1 pins the centre, k = (n+1)/2 is the plain
    filter.  Accepted by ``apply_filter`` like a ``FilterSpec``."""

    family: str
    k: int
    strategy: DirectionalStrategy = field(default_factory=DirectionalStrategy.exact)
    p: float = 2.0
    window: int = 3
    acwddf: Optional[AcwddfParams] = None  # always None (FilterSpec field parity)

    def __post_init__(self) -> None:
        if self.family not in CW_FAMILIES:
            raise ValueError(f"unknown centre-weighted family {self.family!r} (choose from {CW_FAMILIES})")
        if not self.p >= 1.0:
            raise ValueError(f"Minkowski order must be >= 1, got {self.p}")
        if self.window < 3 or self.window % 2 == 0:
            raise ValueError(f"window side must be odd and >= 3, got {self.window}")
        if self.acwddf is not None:
            raise ValueError("centre-weighted specs carry no acwddf parameters")
        center_weight(self.window * self.window, self.k)  # validates k

    @property
    def name(self) -> str:
        out = [self.family, f"k={self.k}"]
        if self.family == "cwddf":
            out.append(self.strategy.token)
            if self.strategy.kind == "minimax":
                out.append(f"q={self.strategy.q}")
        if self.p != 2.0:
            out.append(f"p={_num(self.p)}")
        if self.window != 3:
            out.append(f"window={self.window}")
        return ":".join(out)

    def __str__(self) -> str:
        return self.name


def _num(x: float) -> str:
    x = float(x)
    return str(int(x)) if x == int(x) else repr(x)


_KEYS = ("q", "p", "window", "slope", "intercept", "lambda", "t")


def parse_filter_spec(text: str) -> FilterSpec:
    """Parse ``family[:strategy][:key=value...]`` (e.g. ``acwddf:rgb:lambda=2:T=10.8``)."""
    tokens = [t.strip() for t in text.strip().split(":")]
    tokens = [t for t in tokens if t]
    if not tokens:
        raise ValueError("empty filter spec")
    family = tokens[0].lower()
    if family not in FAMILIES:
        raise ValueError(f"unknown filter family {family!r} in spec {text!r}")
    kind = "exact"
    values: dict = {}
    for tok in tokens[1:]:
        if "=" in tok:
            k, _, v = tok.partition("=")
            values[k.strip().lower()] = v.strip()
        elif tok.lower() in ("exact", "minimax", "rgb"):
            kind = tok.lower()
        else:
            raise ValueError(f"unrecognized token {tok!r} in spec {text!r}")
    unknown = sorted(set(values) - set(_KEYS))
    if unknown:
        raise ValueError(f"unknown keys {unknown} in spec {text!r}")
    try:
        q = int(values.get("q", 4))
        p = float(values.get("p", 2.0))
        window = int(values.get("window", 3))
        slope = float(values.get("slope", CALIBRATION_SLOPE))
        intercept = float(values.get("intercept", CALIBRATION_INTERCEPT))
        lam = int(values.get("lambda", 2))
        threshold = float(values.get("t", 10.8))
    except ValueError as exc:
        raise ValueError(f"bad value in spec {text!r}: {exc}") from None
    if kind == "minimax":
        strategy = DirectionalStrategy.minimax(q)
    elif kind == "rgb":
        strategy = DirectionalStrategy.chromaticity_calibrated(slope, intercept)
    else:
        strategy = DirectionalStrategy.exact()
    acw = AcwddfParams(lam, threshold, p) if family == "acwddf" else None
    return FilterSpec(family=family, strategy=strategy, p=p, window=window, acwddf=acw)
