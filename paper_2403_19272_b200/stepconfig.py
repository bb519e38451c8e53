"""StepConfig / StepReport: identical fields, defaults and validation to the
reference (pkg/src/clothsim/stepper.py:43-92), so configs and harnesses port
unchanged."""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class StepConfig:
    h: float = 1.0 / 150.0
    eps_initial: float = 1e-3
    eps_inner: float = 5e-2
    eps_outer: float = 1e-3
    eps_toi: float = 0.1
    alpha: float = 0.8
    ndb_k: float = 0.0              # 0 -> mean elastic weight
    ndb_base: float = 2.0
    dbb_kappa: float = 0.0          # 0 -> matched to ndb_k at d_hat/2
    iteration_cap: int = 0          # max inner LG iterations per step, 0 = unlimited
    barrier_mode: str = "ndb"
    d_hat: float = 1e-3
    samples: int = 3
    smoothing_iterations: int = 32  # Jacobi updates per inner iteration (16 rank-2 steps)
    omega: float = 0.0
    gravity: tuple = (0.0, 0.0, -9.8)
    warm_start_cap: int = 10
    inner_cap: int = 10
    outer_cap: int = 40
    rf_iterations: int = 30
    rf_tolerance: float = 1e-10
    delta_f_cap: float = 1e6
    r_bar: int = 120
    r: int = 30
    verify: bool = False
    # opt-in (not the reference's smoother; SPEC.md:407 lists Chebyshev as a non-goal):
    # "chebyshev" replaces the rank-2 A-Jacobi updates by Chebyshev-accelerated Jacobi
    # iterations, one fused SELL pass each; "ajacobi" (default) is the parity path
    smoother: str = "ajacobi"

    def __post_init__(self):
        if self.h <= 0 or not (0 < self.alpha < 1):
            raise ValueError("need h > 0 and 0 < alpha < 1")
        for name in ("eps_initial", "eps_inner", "eps_outer", "eps_toi", "d_hat"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.barrier_mode not in ("ndb", "dbb"):
            raise ValueError("barrier_mode must be 'ndb' or 'dbb'")
        if self.smoother not in ("ajacobi", "chebyshev"):
            raise ValueError("smoother must be 'ajacobi' or 'chebyshev'")


@dataclass
class StepReport:
    lg_iterations: int = 0
    outer_loops: int = 0
    toi_exit: float = 1.0
    rf_triggered: bool = False
    penetration_free: bool = True
    active_pairs: int = 0
    full_ccd_calls: int = 0
    partial_ccd_calls: int = 0
    cap_hit: bool = False
    timings: dict = field(default_factory=dict)
