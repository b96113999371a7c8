"""Linear iteration cost model (mirror of `pkg/src/relsim/cost_model.py:23-58, 134-147`).

Prefill duration is linear in uncached tokens, decode duration in the number
of decoding requests.  The device kernels evaluate exactly these two
expressions (one rounded multiply, one rounded add; no FMA).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path


class FitError(ValueError):
    """Calibration samples are insufficient or degenerate."""


@dataclass(frozen=True)
class LinearCostModel:
    alpha_p: float  # s per uncached prefill token
    beta_p: float   # s, prefill intercept
    alpha_d: float  # s per decoding request
    beta_d: float   # s, decode intercept
    clamped: bool = False

    def __post_init__(self):
        if min(self.alpha_p, self.beta_p, self.alpha_d, self.beta_d) < 0:
            raise ValueError("cost model coefficients must be non-negative")


def predict_prefill(model: LinearCostModel, uncached_tokens: int) -> float:
    if uncached_tokens < 0:
        raise ValueError("uncached_tokens must be non-negative")
    return model.alpha_p * uncached_tokens + model.beta_p


def predict_decode(model: LinearCostModel, num_requests: int) -> float:
    if num_requests < 0:
        raise ValueError("num_requests must be non-negative")
    return model.alpha_d * num_requests + model.beta_d


#: World-model presets (cost_model.py:134-138).  "Llama-2-13B" in BASELINE.json
#: maps to opt-13b-like (the only 13B preset), "Llama-2-70B" to llama-70b-like.
WORLD_PRESETS = {
    "opt-13b-like": LinearCostModel(1.0e-4, 0.020, 3.0e-4, 0.020),
    "qwen-32b-like": LinearCostModel(2.2e-4, 0.030, 6.0e-4, 0.030),
    "llama-70b-like": LinearCostModel(5.0e-4, 0.050, 1.2e-3, 0.050),
}


def world_preset(name: str) -> LinearCostModel:
    try:
        return WORLD_PRESETS[name]
    except KeyError:
        raise ValueError(
            f"unknown world model preset {name!r}; available: {sorted(WORLD_PRESETS)}"
        ) from None


def save_model(model: LinearCostModel, path: str | Path) -> None:
    Path(path).write_text(json.dumps({"alpha_p": model.alpha_p, "beta_p": model.beta_p,
                                      "alpha_d": model.alpha_d, "beta_d": model.beta_d},
                                     indent=2) + "\n")


def load_model(path: str | Path) -> LinearCostModel:
    d = json.loads(Path(path).read_text())
    return LinearCostModel(d["alpha_p"], d["beta_p"], d["alpha_d"], d["beta_d"])
