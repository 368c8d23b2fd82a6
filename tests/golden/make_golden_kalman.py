"""Generate tests/golden/kalman_ref.npz: the REAL reference's Kalman filter
NLL and leaf gradients (make_kalman + Graph::backward, dl/models.hpp:272-369)
plus the reference test oracle's dense joint-Gaussian NLL
(proj/tests/kalman_oracle.hpp:16-79), through oracle/_ref/libdla_ref.so
(TEST INFRASTRUCTURE, compiled from /root/reference by oracle/Makefile).

Cases: the scalar random walk with its hand value (proj/tests/
test_models.cpp:187-197), the h = d = 2, T = 5 / T = 4 shapes of the
reference's own recursive-vs-dense and FD tests (:199-241), and larger blocks
up to the kernel's h, d <= 32 limit.  Inputs are stored (small).

    python tests/golden/make_golden_kalman.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

CASES = [(2, 2, 5, 131), (2, 2, 4, 137), (4, 3, 20, 5), (3, 5, 10, 9), (8, 8, 64, 7), (16, 4, 30, 11),
         (1, 1, 200, 4), (32, 32, 12, 5), (6, 2, 128, 13)]
NAMES = ("a", "b", "sh", "sv", "mu0", "s0", "obs")


def main():
    O.build(ref=True)
    out = {}
    one, zero = np.ones((1, 1)), np.zeros((1, 1))
    cases = [("walk", (one, one, one, one, zero, one, np.zeros((2, 1))))]
    for h, d, T, seed in CASES:
        cases.append((f"h{h}d{d}T{T}", O.random_kalman(O.rng(seed), h, d, T)))
    for name, m in cases:
        nll, grads, joint = O.kalman_ref(*m)
        for k, v in zip(NAMES, m):
            out[f"{name}/in/{k}"] = v
        out[f"{name}/nll"] = np.array(nll)
        out[f"{name}/joint"] = np.array(joint)
        for k, v in zip(NAMES, grads):
            out[f"{name}/grad/{k}"] = v
        print(f"{name}: nll {nll!r} joint {joint!r}")
    out["cases"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "kalman_ref.npz"), **out)


if __name__ == "__main__":
    main()
