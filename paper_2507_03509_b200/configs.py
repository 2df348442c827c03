"""BASELINE.json workloads (configs[0..4]) as code + channel parameters.

Codes come from the seeded multi-edge-style generator (csrc/code.cpp,
``generate_met``); sizes follow BASELINE.json literally with round-half-up
class counts and M = round(N * (1 - R)).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

CODE_SEED = 2507_03509  # fixed generator seed for every BASELINE code
FRAME_SEED = 0x5EED_2507


@dataclass(frozen=True)
class Workload:
    name: str
    n_vars: int
    n_checks: int
    frac_deg1: float
    degrees: Tuple[int, ...]
    probs: Tuple[float, ...]
    frames: int
    d_max: int
    betas: Tuple[float, ...]
    # > 0: the two-edge-type construction with a core code (generate_met_core,
    # ext_degree type-2 edges per extension check; `degrees` / `probs` are
    # the core variables' type-1 degrees) instead of the BASELINE generator
    ext_degree: int = 0

    def make_code(self):
        from .decoder import generate_met, generate_met_core
        if self.ext_degree:
            n1 = int(self.frac_deg1 * self.n_vars + 0.5)
            return generate_met_core(self.n_vars, self.n_checks, n1, self.degrees, self.probs, self.ext_degree,
                                     CODE_SEED)
        return generate_met(self.n_vars, self.n_checks, self.frac_deg1, self.degrees, self.probs, CODE_SEED)


def _m(n: int, rate: float) -> int:
    return int(n * (1.0 - rate) + 0.5)


WORKLOADS = {
    # configs[0]: small CPU-oracle workload
    "cfg1": Workload("cfg1_r0.1_n8192", 8192, _m(8192, 0.1), 0.75, (3, 6, 12), (0.5, 0.3, 0.2), 16, 200, (0.95,)),
    # configs[1]: the headline single-GPU workload
    "cfg2": Workload("cfg2_r0.1_n2^20", 1 << 20, _m(1 << 20, 0.1), 0.75, (3, 6, 12), (0.5, 0.3, 0.2), 64, 500,
                     (0.92, 0.94, 0.96, 0.98, 0.99)),
    # configs[2]: ultra-low rate
    "cfg3": Workload("cfg3_r0.02_n2^20", 1 << 20, _m(1 << 20, 0.02), 0.90, (2, 3, 20), (0.3, 0.4, 0.3), 32, 500,
                     (0.98,)),
    # configs[3]: frame-parallel sweep on the config-2 code
    "cfg4": Workload("cfg4_r0.1_n2^20_sweep", 1 << 20, _m(1 << 20, 0.1), 0.75, (3, 6, 12), (0.5, 0.3, 0.2), 4096,
                     500, (0.95,)),
    # configs[4]: mixed-SNR streaming, beta ~ U[0.92, 1.0] per frame
    "cfg5": Workload("cfg5_r0.05_n2^21_stream", 1 << 21, _m(1 << 21, 0.05), 0.80, (3, 8, 16), (0.5, 0.3, 0.2),
                     8192, 500, (0.92, 1.0)),
    # a code family whose FER falls below 1 (the BASELINE
    # construction's never does): rate 0.1, 70% degree-1 variables on
    # extension checks with 2 core edges each, core variables of type-1
    # degree 2 / 3 on a core code (check degrees 3 / 4)
    "met": Workload("met_r0.1_n2^20", 1 << 20, _m(1 << 20, 0.1), 0.70, (2, 3), (0.5, 0.5), 64, 500,
                    (0.84, 0.85, 0.86, 0.87, 0.88, 0.89, 0.90), ext_degree=2),
    "met_s": Workload("met_r0.1_n8192", 8192, _m(8192, 0.1), 0.70, (2, 3), (0.5, 0.5), 16, 200, (0.7, 0.8, 0.9),
                      ext_degree=2),
}
