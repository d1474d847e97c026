"""Closed-form batch-size hyperparameter scaling (SPEC.md `hparam_scaling`,
340-398; reference src/hparam_scaling.cpp:32-65). Host math for the
`scale-hparams` CLI subcommand; never on the step path."""
from __future__ import annotations

import math
from dataclasses import dataclass

THEORY_SQRT, HEURISTIC_LINEAR = "theory_sqrt", "heuristic_linear"


def scale_lr(eps: float, k: float, rule: str = THEORY_SQRT) -> float:
    """eps * sqrt(k) (theory) or eps * k (heuristic) (hparam_scaling.cpp:32-36)."""
    if not eps > 0:
        raise ValueError("scale_lr: lr must be positive")
    if not k > 0:
        raise ValueError("scale_lr: k must be positive")
    if rule == THEORY_SQRT:
        return eps * math.sqrt(k)
    if rule == HEURISTIC_LINEAR:
        return eps * k
    raise ValueError(f"scale_lr: unknown rule {rule!r}")


def scale_weight_decay_exact(eps: float, omega: float, k: float) -> float:
    """omega' = (1 - (1 - eps*omega)^k) / (sqrt(k) * eps) (hparam_scaling.cpp:38-46):
    k decayed steps at (eps, omega) equal one at (sqrt(k) eps, omega')."""
    if not k > 0:
        raise ValueError("scale_weight_decay_exact: k must be positive")
    if not eps * omega < 1:
        raise ValueError(f"scale_weight_decay_exact: lr*weight_decay = {eps * omega} must be < 1")
    return (1.0 - math.pow(1.0 - eps * omega, k)) / (math.sqrt(k) * eps)


def scale_weight_decay_approx(omega: float, k: float) -> float:
    """omega' ~= sqrt(k) * omega, the eps -> 0 limit (hparam_scaling.cpp:48-51)."""
    if not k > 0:
        raise ValueError("scale_weight_decay_approx: k must be positive")
    return math.sqrt(k) * omega


@dataclass
class ScalePlan:
    k: float
    eps: float
    omega: float
    rule: str
    eps_new: float
    omega_exact: float
    omega_approx: float
    omega_practical: float  # §5: "I used omega' = omega = 0.0005 for all experiments"


def make_scale_plan(eps: float, omega: float, k: float, rule: str = THEORY_SQRT) -> ScalePlan:
    """hparam_scaling.cpp:53-65."""
    return ScalePlan(k, eps, omega, rule, scale_lr(eps, k, rule), scale_weight_decay_exact(eps, omega, k),
                     scale_weight_decay_approx(omega, k), omega)
