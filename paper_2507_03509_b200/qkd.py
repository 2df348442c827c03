"""CV-QKD key-rate accounting around the decoder: Eq. (1)-(3) of the paper
 and the beta optimiser (PAPER.md "for each capture beta
was optimised"; SPEC.md qkd-metrics module).

The reference's own implementation of this module (qkd_metrics.cpp) is not
in the mounted reference tree, so this follows the SPEC's
stated closed forms and is pinned by the SPEC's worked examples
(tests/test_qkd.py):

* trusted-receiver Gaussian model: V = V_A + 1, T = 10^(-alpha d / 10),
  chi_line = 1/T - 1 + xi, chi_het = (1 + (1 - eta) + 2 nu_el) / eta,
  chi_hom = ((1 - eta) + nu_el) / eta, chi_tot = chi_line + chi_det / T;
* I_AB = (mu / 2) log2((V + chi_tot) / (1 + chi_tot));
* chi_BE = g(nu1) + g(nu2) - g(nu3) - g(nu4) (entangling-cloner bound);
* Delta_n = 7 sqrt(log2(2 / eps_bar) / n) + (2 / n) log2(1 / eps_pa);
* SKR = (1 - FER)(beta I_AB - chi_BE - Delta_n)         (Eq. 1)
* K = N R (1 - FER) / D_bar                              (Eq. 2)
* SKR_dec = N (1 - FER)(beta I_AB - chi_BE - Delta_n) / (D_bar mu)   (Eq. 3)

Pure host-side functions (no device code): they turn the decoder's FER and
mean iterations (bench.py, scripts/vnr_pce_sweep.py) into key rates.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Iterable, List, Optional, Tuple


@dataclass(frozen=True)
class QkdSystemParams:
    """SPEC.md qkd-metrics QkdSystemParams.  Defaults: the paper's
    simulation operating point (PAPER.md "Simulations": eta = 0.4, nu_el =
    0.01, xi = 0.001, 80 km at 0.2 dB/km, heterodyne, N_privacy = 1e8)."""
    distance_km: float = 80.0
    loss_db_per_km: float = 0.2
    eta: float = 0.4
    nu_el: float = 0.01
    xi: float = 0.001
    v_a: float = 1.0
    mu: int = 2                 # 1 homodyne, 2 heterodyne
    n_privacy: float = 1e8
    eps_bar: float = 1e-10
    eps_pa: float = 1e-10
    f_rep: Optional[float] = None
    transmittance_override: Optional[float] = None  # T directly (tests / back-to-back)

    @property
    def transmittance(self) -> float:
        if self.transmittance_override is not None:
            return self.transmittance_override
        return 10.0 ** (-self.loss_db_per_km * self.distance_km / 10.0)

    def validate(self) -> None:
        T = self.transmittance
        if not (0.0 < T <= 1.0):
            raise ValueError("qkd: transmittance must lie in (0, 1]")
        if not (0.0 < self.eta <= 1.0):
            raise ValueError("qkd: eta must lie in (0, 1]")
        if self.nu_el < 0 or self.xi < 0:
            raise ValueError("qkd: nu_el and xi must be >= 0")
        if not self.v_a > 0:
            raise ValueError("qkd: V_A must be positive")
        if self.mu not in (1, 2):
            raise ValueError("qkd: mu must be 1 (homodyne) or 2 (heterodyne)")


@dataclass
class SkrBreakdown:
    """SPEC.md SkrBreakdown (per-pulse quantities in bits)."""
    i_ab: float
    chi_be: float
    delta_n: float
    fer: float
    beta: float
    skr: float
    k_throughput: Optional[float] = None
    skr_dec: Optional[float] = None
    negative: bool = False   # beta I_AB - chi_BE - Delta_n < 0 (reported, not clipped)


def _chis(p: QkdSystemParams):
    T = p.transmittance
    chi_line = 1.0 / T - 1.0 + p.xi
    chi_det = ((1.0 + (1.0 - p.eta) + 2.0 * p.nu_el) / p.eta if p.mu == 2
               else ((1.0 - p.eta) + p.nu_el) / p.eta)
    return T, chi_line, chi_det, chi_line + chi_det / T


def mutual_information(p: QkdSystemParams) -> float:
    """I_AB in bits per pulse (SPEC mutual_information)."""
    p.validate()
    _, _, _, chi_tot = _chis(p)
    V = p.v_a + 1.0
    return 0.5 * p.mu * math.log2((V + chi_tot) / (1.0 + chi_tot))


def solve_va_for_iab(target_iab: float, p: QkdSystemParams) -> float:
    """V_A with mutual_information(p with v_a = V_A) = target (closed-form
    inversion; PAPER.md "V_A chosen such that I_AB = R / beta")."""
    if not target_iab > 0:
        raise ValueError("qkd: target I_AB must be positive")
    _, _, _, chi_tot = _chis(p)
    ratio = 2.0 ** (2.0 * target_iab / p.mu)
    if not math.isfinite(ratio):
        raise ValueError("qkd: target I_AB out of numeric range")
    V = ratio * (1.0 + chi_tot) - chi_tot
    va = V - 1.0
    if not va > 0:
        raise ValueError("qkd: no positive V_A reaches the target I_AB")
    return va


def g_entropy(x: float) -> float:
    """g(x) = ((x+1)/2) log2((x+1)/2) - ((x-1)/2) log2((x-1)/2), g(1) = 0."""
    if x < 1.0 - 1e-9:
        raise ValueError(f"qkd: symplectic eigenvalue {x} < 1 (unphysical parameters)")
    a = (x + 1.0) / 2.0
    b = (x - 1.0) / 2.0
    return a * math.log2(a) - (b * math.log2(b) if b > 0 else 0.0)


def _sym_eigs(A: float, B: float) -> Tuple[float, float]:
    disc = max(A * A - 4.0 * B, 0.0)
    r = math.sqrt(disc)
    return math.sqrt(max(0.5 * (A + r), 0.0)), math.sqrt(max(0.5 * (A - r), 0.0))


def holevo_bound(p: QkdSystemParams) -> float:
    """chi_BE in bits per pulse (SPEC holevo_bound; entangling-cloner
    model, trusted receiver noise, heterodyne or homodyne)."""
    p.validate()
    T, chi_line, chi_det, chi_tot = _chis(p)
    V = p.v_a + 1.0
    A = V * V * (1.0 - 2.0 * T) + 2.0 * T + T * T * (V + chi_line) ** 2
    B = T * T * (V * chi_line + 1.0) ** 2
    n1, n2 = _sym_eigs(A, B)
    sB = math.sqrt(B)
    den = T * (V + chi_tot)
    A3 = (A * chi_det + V * sB + T * (V + chi_line)) / den
    B3 = sB * (V + sB * chi_det) / den
    n3, n4 = _sym_eigs(A3, B3)
    nus = [max(n, 1.0) if n > 1.0 - 1e-9 else n for n in (n1, n2, n3, n4)]
    return g_entropy(nus[0]) + g_entropy(nus[1]) - g_entropy(nus[2]) - g_entropy(nus[3])


def finite_size_penalty(p: QkdSystemParams) -> float:
    """Delta_n (SPEC finite_size_penalty)."""
    if p.n_privacy < 1e4:
        raise ValueError("qkd: n_privacy must be >= 1e4")
    n = p.n_privacy
    return 7.0 * math.sqrt(math.log2(2.0 / p.eps_bar) / n) + (2.0 / n) * math.log2(1.0 / p.eps_pa)


def _check_beta_fer(beta: float, fer: float) -> None:
    if not (0.0 <= fer <= 1.0):
        raise ValueError("qkd: FER must lie in [0, 1]")
    if not (0.0 < beta <= 1.0):
        raise ValueError("qkd: beta must lie in (0, 1]")


def eq1(beta: float, fer: float, i_ab: float, chi_be: float, delta_n: float) -> float:
    """Eq. (1) on given terms."""
    _check_beta_fer(beta, fer)
    return (1.0 - fer) * (beta * i_ab - chi_be - delta_n)


def eq3(n: float, d_bar: float, mu: int, fer: float, core: float) -> float:
    """Eq. (3) on given terms; core = beta I_AB - chi_BE - Delta_n."""
    if d_bar < 1.0:
        raise ValueError("qkd: D_bar must be >= 1")
    return n / (d_bar * mu) * (1.0 - fer) * core


def skr(p: QkdSystemParams, beta: float, fer: float) -> SkrBreakdown:
    """Eq. (1): SKR = (1 - FER)(beta I_AB - chi_BE - Delta_n), bits/pulse."""
    _check_beta_fer(beta, fer)
    i_ab, chi, dn = mutual_information(p), holevo_bound(p), finite_size_penalty(p)
    core = beta * i_ab - chi - dn
    return SkrBreakdown(i_ab=i_ab, chi_be=chi, delta_n=dn, fer=fer, beta=beta, skr=(1.0 - fer) * core,
                        negative=core < 0)


def decoder_throughput(n: float, d_bar: float, rate: float, fer: float) -> float:
    """Eq. (2): K = N R (1 - FER) / D_bar, bits per iteration latency t."""
    if d_bar < 1.0:
        raise ValueError("qkd: D_bar must be >= 1")
    return n / d_bar * rate * (1.0 - fer)


def skr_dec(p: QkdSystemParams, beta: float, fer: float, n: float, d_bar: float) -> float:
    """Eq. (3): SKR_dec = N (1 - FER)(beta I_AB - chi_BE - Delta_n) / (D_bar mu)."""
    b = skr(p, beta, fer)
    if d_bar < 1.0:
        raise ValueError("qkd: D_bar must be >= 1")
    return n / (d_bar * p.mu) * b.skr


def operating_point(rate: float, beta: float, p: Optional[QkdSystemParams] = None) -> QkdSystemParams:
    """The paper's simulation convention: V_A such that I_AB = R / beta."""
    p = p or QkdSystemParams()
    return replace(p, v_a=solve_va_for_iab(rate / beta, p))


def evaluate(rate: float, beta: float, fer: float, n: float, d_bar: float,
             p: Optional[QkdSystemParams] = None) -> SkrBreakdown:
    """SKR, K and SKR_dec of one sweep point (beta, FER, D_bar) at the
    paper's operating-point convention."""
    q = operating_point(rate, beta, p)
    b = skr(q, beta, fer)
    b.k_throughput = decoder_throughput(n, d_bar, rate, fer)
    b.skr_dec = n / (d_bar * q.mu) * b.skr
    return b


@dataclass(frozen=True)
class SweepRecord:
    beta: float
    skr: float
    skr_dec: float


def optimize_beta(records: Iterable[SweepRecord]) -> Tuple[float, float]:
    """(beta_opt for SKR, beta_opt for SKR_dec): argmax over the sweep grid,
    ties broken toward the lower beta (SPEC optimize_beta)."""
    recs: List[SweepRecord] = sorted(records, key=lambda r: r.beta)
    if not recs:
        raise ValueError("qkd: optimize_beta needs at least one record")
    best_skr = max(recs, key=lambda r: (r.skr, -r.beta))
    best_dec = max(recs, key=lambda r: (r.skr_dec, -r.beta))
    return best_skr.beta, best_dec.beta
