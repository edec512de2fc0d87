import numpy as np


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(a - b)
    s = max(np.linalg.norm(b), 1e-300)
    return d / s


def rand(n, seed=42):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)
