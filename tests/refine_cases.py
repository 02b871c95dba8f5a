"""The exhaustive Eq. 3-5 case set of reference tests/test_acceptance.py:327-373."""
import numpy as np

REGULAR_TYPES = (0x99, 0x66, 0x33, 0xCC, 0x0F, 0xF0)


def refine_cases(eps=0.1):
    below, above = eps * 0.5, eps * 2.0
    patterns = [np.full(8, below), np.full(8, above)]
    alt = np.full(8, below)
    alt[1::2] = above
    patterns.append(alt)
    patterns.append(alt[::-1].copy())
    rng = np.random.default_rng(42)
    patterns.append(rng.choice([below, above, eps, -below, -above], size=8))
    for t_curr in range(256):
        prev_set = {t_curr, t_curr ^ 0x01, t_curr ^ 0x0B, t_curr ^ 0x0F}
        prev_set.update(REGULAR_TYPES)
        for t_prev in sorted(prev_set):
            for corners in patterns:
                yield t_curr, t_prev, corners
