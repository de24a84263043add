"""Weight vectors at the edges of f64, shared by the reference pins
(test_ref_pins.py) and the GPU parity tests."""
import numpy as np


def extreme_cases():
    """Magnitudes at the edges of f64: totals >= 1e300 (the guarded
    compensated add), an infinite total (weights.hpp:32-46 accepts it; every
    item is then light), subnormal weights."""
    rng = np.random.default_rng(8)
    return [rng.random(1000) * 1e305 + 1e304,
            np.full(1000, 1e306),
            np.concatenate([np.full(500, 1.7e308), rng.random(700) + 0.1]),
            10.0 ** rng.uniform(-323, -300, 3000),
            np.where(rng.random(5000) < 0.5, 5e-324 * rng.integers(1, 1000, 5000), 1.0),
            10.0 ** rng.uniform(-300, 300, 5000)]
