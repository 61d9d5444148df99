"""Reader for the small text fixtures under tests/golden/ (name | values, '#' comments)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, vals = line.split("|", 1)
            out[key.strip()] = np.array([float(v) for v in vals.split()])
    return out
